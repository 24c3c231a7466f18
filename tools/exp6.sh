S=gpurun_out/exp6_sweep.txt
run() { lab=$1; g=$2; inf=$3; shift 3; env "$@" bash tools/sweep.sh "$lab" --group $g --inflight $inf --steps 300 --no-check >> $S 2>&1; }
bash tools/sweep.sh "single" --inflight 6 --steps 300 --no-check >> $S 2>&1
run g3i2_w8 3 2 DCI_TMA_WARPS=8
run g3i2_w8_prio 3 2 DCI_TMA_WARPS=8 DCI_SAMPLE_PRIO=1
run g3i2_w8_nohint 3 2 DCI_TMA_WARPS=8 DCI_TMA_HINT=0
run g2i4_w8 2 4 DCI_TMA_WARPS=8
run g2i4_w8_prio 2 4 DCI_TMA_WARPS=8 DCI_SAMPLE_PRIO=1
run g4i3_w8 4 3 DCI_TMA_WARPS=8
run g1i6_w8 1 6 DCI_TMA_WARPS=8
run g1i6_w8_prio 1 6 DCI_TMA_WARPS=8 DCI_SAMPLE_PRIO=1
run g6i2_w8_prio 6 2 DCI_TMA_WARPS=8 DCI_SAMPLE_PRIO=1
cat $S
