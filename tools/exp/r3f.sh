# session 3: bench line with batch latency + host memory; multireader probe at the visible reader count
mkdir -p gpurun_out/r3f; rm -rf gpurun_out/r3f/*
timeout 900 python -m pytest tests/test_gpu_bench.py -q -x 2>&1 | tail -3 > gpurun_out/r3f/tests.txt
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 > gpurun_out/r3f/bench_M1.json 2> gpurun_out/r3f/bench_M1.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r3f/bench_M2_k20.json 2> gpurun_out/r3f/bench_M2_k20.log
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 > gpurun_out/r3f/bench_M3.json 2> gpurun_out/r3f/bench_M3.log
bash tools/probe/run_multireader.sh 8 > gpurun_out/r3f/multireader.log 2>&1
cp profiles/hostlink_*reader.json gpurun_out/r3f/ 2>/dev/null
cat gpurun_out/r3f/tests.txt
for c in M1 M2_k20 M3; do python -c "
import json; d=json.load(open('gpurun_out/r3f/bench_$c.json')); print('$c', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), d['roofline']['frac'], d['latency'], d['host_memory'])"; done
tail -5 gpurun_out/r3f/multireader.log
