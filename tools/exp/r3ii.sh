# session 3: M5 split sweep (F3) under the final defaults (groups of 32, node-sweep gathers)
mkdir -p gpurun_out/r3ii; rm -rf gpurun_out/r3ii/*
for fan in 2,2,2 8,4,2 15,10,5; do
  t=$(echo $fan | tr , _)
  timeout 900 python bench.py --config M5 --fanouts $fan --steps 64 --warmup 8 --repeats 3 --no-cpu-baseline --no-check --no-latency --no-aggregate > gpurun_out/r3ii/m5_${t}_eq1.json 2> /dev/null
  for r in 0.0 0.1 0.2 0.3 0.5 0.7 1.0; do
    timeout 900 python bench.py --config M5 --fanouts $fan --ratio $r --steps 64 --warmup 8 --repeats 3 --no-cpu-baseline --no-check --no-latency --no-aggregate > gpurun_out/r3ii/m5_${t}_r$r.json 2> /dev/null
  done
done
for f in gpurun_out/r3ii/*.json; do python -c "
import json; d=json.load(open('$f')); s=d['stats']; print('$f', round(d['value']/1e6,3), round(s['c_adj']/(s['c_adj']+s['c_feat']),3), round(s['adj_hit_rate'],3), round(s['feat_hit_rate'],3))" 2>/dev/null; done
