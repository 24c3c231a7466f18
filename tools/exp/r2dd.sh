mkdir -p gpurun_out/r2dd
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2dd/bench_M2.json 2> gpurun_out/r2dd/bench_M2.log
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2dd/bench_M1.json 2> gpurun_out/r2dd/bench_M1.log
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2dd/bench_M3.json 2> gpurun_out/r2dd/bench_M3.log
timeout 900 python -m pytest tests/test_gpu_bench.py -q -x 2>&1 | tail -3 > gpurun_out/r2dd/tests_bench.txt
