# session 3: GroupCall (fixed arguments marshalled once) -- host time, region time, parity, M2 bench
mkdir -p gpurun_out/r3t; rm -rf gpurun_out/r3t/*
python tools/exp/host_overhead.py > gpurun_out/r3t/host_overhead.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_many.py tests/test_gpu_bench.py -q -x 2>&1 | tail -2 > gpurun_out/r3t/tests.txt
for i in 1 2 3; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3t/m2_$i.json 2> /dev/null; done
cat gpurun_out/r3t/host_overhead.txt gpurun_out/r3t/tests.txt
for f in gpurun_out/r3t/m2_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), d['stats']['host_enqueue_ms_per_step'])"; done
