mkdir -p gpurun_out/r2ff
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -k "bench_launch or m2_reddit" 2>&1 | tail -5 > gpurun_out/r2ff/tests.txt
