# session 3: M3 (host-link bound) in groups of 20 -- the node-sweep gather reads each miss row once per group
mkdir -p gpurun_out/r3x; rm -rf gpurun_out/r3x/*
for i in 1 2; do
  timeout 900 python bench.py --config M3 --steps 40 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3x/m3_single_$i.json 2> /dev/null
  timeout 900 python bench.py --config M3 --steps 40 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate --group 20 --inflight 2 > gpurun_out/r3x/m3_g20_$i.json 2> /dev/null
  timeout 900 python bench.py --config M3 --steps 40 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate --group 20 --inflight 1 > gpurun_out/r3x/m3_g20i1_$i.json 2> /dev/null
done
timeout 900 python bench.py --config M3 --steps 40 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate --group 32 --inflight 2 > gpurun_out/r3x/m3_g32.json 2> /dev/null
for f in gpurun_out/r3x/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; h=d['host_link']; print('$f', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), r.get('gather_kernels'), round(h.get('host_payload_GBps') or 0,1), d['stats']['feat_hit_rate'])"; done
