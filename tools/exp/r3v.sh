# session 3: GroupCall.host in the e2e leg; GPU tests of the group path and the bench line
mkdir -p gpurun_out/r3v; rm -rf gpurun_out/r3v/*
timeout 1200 python -m pytest tests/test_gpu_many.py tests/test_gpu_bench.py -q -x 2>&1 | tail -2 > gpurun_out/r3v/tests.txt
for i in 1 2 3; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3v/m2_$i.json 2> /dev/null; done
cat gpurun_out/r3v/tests.txt
for f in gpurun_out/r3v/m2_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), d['parity_check'] if 'parity_check' in d else '')"; done
