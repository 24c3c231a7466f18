mkdir -p gpurun_out/r2kk
for g in 0 4 8 16; do
timeout 900 python bench.py --config M3 --steps 40 --warmup 8 --group $g --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2kk/M3_g$g.json 2> gpurun_out/r2kk/M3_g$g.log
done
for inf in 4 8; do
timeout 900 python bench.py --config M3 --steps 40 --warmup 8 --group 0 --inflight $inf --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2kk/M3_g0_i$inf.json 2> gpurun_out/r2kk/M3_g0_i$inf.log
done
