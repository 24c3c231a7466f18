# session 3: F3 presample-count sweep on papers100M-shaped graphs under the final defaults (groups of 32, node-sweep gathers)
mkdir -p gpurun_out/r3hh; rm -rf gpurun_out/r3hh/*
for n in 8 32 128; do
timeout 900 python bench.py --config M4s --steps 64 --warmup 8 --repeats 3 --no-cpu-baseline --no-check --no-latency --no-aggregate --presample-batches $n > gpurun_out/r3hh/M4s_pre$n.json 2> gpurun_out/r3hh/M4s_pre$n.log
done
for n in 8 64 256; do
timeout 2400 python bench.py --config M4 --steps 64 --warmup 8 --repeats 3 --no-cpu-baseline --no-check --no-latency --no-aggregate --presample-batches $n > gpurun_out/r3hh/M4_pre$n.json 2> gpurun_out/r3hh/M4_pre$n.log
done
for f in gpurun_out/r3hh/*.json; do python -c "
import json; d=json.load(open('$f')); s=d['stats']; p=s['preprocess_s']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(s['feat_hit_rate'],3), round(s['adj_hit_rate'],3), round(p['presample'],2), round(p['allocate_fill'],2))"; done
