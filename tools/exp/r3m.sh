# session 3: M4 (111 M nodes, 3.5 GB directory) under the sampler's directory L2 policy: evict-last (0) vs normal (1)
mkdir -p gpurun_out/r3m; rm -rf gpurun_out/r3m/*
for i in 1 2; do
  for c in 1 0; do
    DCI_DIR_POLICY=$c timeout 1200 python bench.py --config M4 --steps 40 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3m/m4_d${c}_$i.json 2> gpurun_out/r3m/m4_d${c}_$i.log
  done
done
for f in gpurun_out/r3m/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(d['roofline']['frac'],3), d['host_link']['request_view']['M_requests_per_s'])"; done
