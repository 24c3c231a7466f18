# session 3: groups of 32 (DCI_MAX_GROUP) vs 20 on the host-resident configs (more batches share each miss row)
mkdir -p gpurun_out/r3cc; rm -rf gpurun_out/r3cc/*
for c in M3 M4s; do
  for g in 20 32; do
    timeout 900 python bench.py --config $c --steps 64 --warmup 8 --group $g --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3cc/${c}_g$g.json 2> /dev/null
  done
done
for g in 20 32; do
  timeout 2400 python bench.py --config M4 --steps 64 --warmup 8 --group $g --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3cc/M4_g$g.json 2> /dev/null
done
for f in gpurun_out/r3cc/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['rows_read_per_row'],3), r.get('gather_kernels'))"; done
