# session 3: M2 with groups of 32 (K = 300 and the driver's K = 20) vs 20
mkdir -p gpurun_out/r3nn; rm -rf gpurun_out/r3nn/*
for g in 20 32; do
  timeout 600 python bench.py --steps 300 --warmup 20 --group $g --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3nn/m2_k300_g$g.json 2> /dev/null
  timeout 600 python bench.py --steps 20 --warmup 5 --group $g --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3nn/m2_k20_g$g.json 2> /dev/null
done
for f in gpurun_out/r3nn/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), d['gpu_launches'])"; done
