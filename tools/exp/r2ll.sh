mkdir -p gpurun_out/r2ll
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 --no-cpu-baseline --no-check > gpurun_out/r2ll/M3.json 2> gpurun_out/r2ll/M3.log
timeout 600 python bench.py --steps 20 --warmup 5 --group 0 --no-cpu-baseline --no-check > gpurun_out/r2ll/M2_g0.json 2> gpurun_out/r2ll/M2_g0.log
timeout 900 python -m pytest tests/test_gpu_bench.py -q -x 2>&1 | tail -3 > gpurun_out/r2ll/tests.txt
