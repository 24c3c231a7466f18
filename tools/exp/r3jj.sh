# session 3: Eq. 1 inputs from group stage times (--eq1-times group) vs the presample's per-batch times
mkdir -p gpurun_out/r3jj; rm -rf gpurun_out/r3jj/*
for fan in 2,2,2 8,4,2 15,10,5; do
  t=$(echo $fan | tr , _)
  for m in presample group; do
    timeout 900 python bench.py --config M5 --fanouts $fan --eq1-times $m --steps 64 --warmup 8 --repeats 3 --no-cpu-baseline --no-check --no-latency --no-aggregate > gpurun_out/r3jj/m5_${t}_$m.json 2> gpurun_out/r3jj/m5_${t}_$m.log
  done
done
for m in presample group; do
  timeout 900 python bench.py --config M4s --eq1-times $m --steps 64 --warmup 8 --no-cpu-baseline --check-light --no-latency --no-aggregate > gpurun_out/r3jj/m4s_$m.json 2> gpurun_out/r3jj/m4s_$m.log
  timeout 2400 python bench.py --config M4 --eq1-times $m --steps 64 --warmup 8 --no-cpu-baseline --check-light --no-latency --no-aggregate > gpurun_out/r3jj/m4_$m.json 2> gpurun_out/r3jj/m4_$m.log
done
for f in gpurun_out/r3jj/*.json; do python -c "
import json; d=json.load(open('$f')); s=d['stats']; print('$f', round(d['value']/1e6,4), round(s['c_adj']/(s['c_adj']+s['c_feat']),3), round(s['adj_hit_rate'],3), round(s['feat_hit_rate'],3), d.get('parity_check',{}).get('bit_exact'))" 2>/dev/null; done
grep -h "Eq. 1 inputs" gpurun_out/r3jj/*.log | head -8
