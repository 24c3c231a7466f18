# session 3: groups in flight (2 vs 3) on the host-resident configs
mkdir -p gpurun_out/r3oo; rm -rf gpurun_out/r3oo/*
for i in 2 3; do
  timeout 900 python bench.py --config M3 --steps 96 --warmup 8 --inflight $i --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3oo/m3_i$i.json 2> /dev/null
  timeout 900 python bench.py --config M4s --steps 96 --warmup 8 --inflight $i --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3oo/m4s_i$i.json 2> /dev/null
done
for f in gpurun_out/r3oo/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4))"; done
