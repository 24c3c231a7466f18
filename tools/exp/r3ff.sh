# session 3: node-sweep gather kind on the host-resident configs: auto (bulk alone / registers beside sampling) vs always bulk vs always registers
mkdir -p gpurun_out/r3ff; rm -rf gpurun_out/r3ff/*
for k in auto tma ldg; do
  DCI_SWEEP_KIND=$k timeout 900 python bench.py --config M3 --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ff/m3_$k.json 2> /dev/null
  DCI_SWEEP_KIND=$k timeout 900 python bench.py --config M4s --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ff/m4s_$k.json 2> /dev/null
done
for k in auto tma; do
  DCI_SWEEP_KIND=$k timeout 2400 python bench.py --config M4 --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ff/m4_$k.json 2> /dev/null
done
for f in gpurun_out/r3ff/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['avg_gather_ms'],2), r.get('gather_kernels'))"; done
