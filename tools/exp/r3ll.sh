# session 3: node-sweep sampling for host-resident adjacency below the cover threshold (DCI_SWEEP_FACTOR: sweep when the hop's frontier total >= factor x N)
mkdir -p gpurun_out/r3ll; rm -rf gpurun_out/r3ll/*
DCI_SWEEP_FACTOR=0.05 timeout 900 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py -q -x 2>&1 | tail -2 > gpurun_out/r3ll/tests.txt
for fct in 1 0.1 0.02; do
  DCI_SWEEP_FACTOR=$fct timeout 900 python bench.py --config M3 --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ll/m3_f$fct.json 2> /dev/null
  DCI_SWEEP_FACTOR=$fct timeout 900 python bench.py --config M4s --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ll/m4s_f$fct.json 2> /dev/null
done
DCI_SWEEP_FACTOR=0.1 timeout 900 python bench.py --config M3 --steps 64 --warmup 8 --check-light --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ll/m3_f0.1_check.json 2> /dev/null
cat gpurun_out/r3ll/tests.txt
for f in gpurun_out/r3ll/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['avg_sample_ms'],3), round(r['avg_gather_ms'],2), d.get('parity_check',{}).get('bit_exact'))"; done
