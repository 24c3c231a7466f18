# session 3: no k_newmask_sweep launch for hops whose frontier capacities cannot reach N
mkdir -p gpurun_out/r3r; rm -rf gpurun_out/r3r/*
timeout 1500 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > gpurun_out/r3r/tests.txt
for i in 1 2 3; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3r/m2_$i.json 2> /dev/null; done
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 --no-cpu-baseline --no-aggregate > gpurun_out/r3r/m1.json 2> /dev/null
bash tools/exp/launches.sh nm --steps 20 --warmup 5; cp gpurun_out/exp/launches_nm.csv gpurun_out/r3r/
cat gpurun_out/r3r/tests.txt
for f in gpurun_out/r3r/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), d['gpu_launches'], (d.get('latency') or {}).get('launches_per_batch'))"; done
