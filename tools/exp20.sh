timeout 600 python bench.py > gpurun_out/bench_M2.json 2> gpurun_out/bench_M2.log
timeout 600 python bench.py --config M1 > gpurun_out/bench_M1.json 2> gpurun_out/bench_M1.log
bash tools/profile.sh r01m > /dev/null 2>&1
cat gpurun_out/bench_M2.json gpurun_out/bench_M1.json
