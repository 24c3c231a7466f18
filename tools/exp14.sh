S=gpurun_out/exp14_sweep.txt
run() { lab=$1; shift; env "$@" bash tools/sweep.sh "$lab" --steps 384 --no-check >> $S 2>&1; }
run pol0 DCI_ELEM_POLICY=0
run pol1 DCI_ELEM_POLICY=1
run pol2 DCI_ELEM_POLICY=2
run pol0b DCI_ELEM_POLICY=0
cat $S
for p in 0 2; do
DCI_ELEM_POLICY=$p ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/exp14_l$p.csv python bench.py --profile-only --steps 24 --warmup 6 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/exp14_l$p.csv 2>/dev/null | head -0
done
