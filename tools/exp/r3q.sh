# session 3: the new switch-matrix cases and the bench-line test
mkdir -p gpurun_out/r3q; rm -rf gpurun_out/r3q/*
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -k "variants" tests/test_gpu_bench.py -q 2>&1 | tail -4 > gpurun_out/r3q/tests.txt
cat gpurun_out/r3q/tests.txt
