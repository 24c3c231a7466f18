mkdir -p gpurun_out/r2w
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2w/bench_M2_k20_$i.json 2> gpurun_out/r2w/bench_M2_k20_$i.log
done
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --no-check > gpurun_out/r2w/bench_M4s.json 2> gpurun_out/r2w/bench_M4s.log
