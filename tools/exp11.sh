timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/exp11_tests.txt
timeout 600 python bench.py > gpurun_out/bench_M2.json 2> gpurun_out/bench_M2.log
bash tools/profile.sh r01g > /dev/null 2>&1
cat gpurun_out/exp11_tests.txt gpurun_out/bench_M2.json
