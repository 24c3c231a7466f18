mkdir -p gpurun_out/r2x
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r2x/tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2x/bench_M2_k20.json 2> gpurun_out/r2x/bench_M2_k20.log
for i in 1 2; do
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --no-check > gpurun_out/r2x/bench_M4s_$i.json 2> gpurun_out/r2x/bench_M4s_$i.log
done
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2x/bench_M3.json 2> gpurun_out/r2x/bench_M3.log
