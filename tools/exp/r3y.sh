# session 3: groups of 20 with node-sweep gathers on the host-resident configs (each miss row read once per group)
mkdir -p gpurun_out/r3y; rm -rf gpurun_out/r3y/*
timeout 900 python bench.py --config M3 --steps 40 --warmup 8 --group 20 --inflight 2 > gpurun_out/r3y/m3_g20_parity.json 2> gpurun_out/r3y/m3_g20_parity.log
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --check-light > gpurun_out/r3y/m4s_g8.json 2> gpurun_out/r3y/m4s_g8.log
DCI_TABLE=dense timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --check-light --group 20 --inflight 2 > gpurun_out/r3y/m4s_g20_dense.json 2> gpurun_out/r3y/m4s_g20_dense.log
DCI_TABLE=dense timeout 1800 python bench.py --config M4 --steps 40 --warmup 8 --no-cpu-baseline --check-light --group 20 --inflight 2 > gpurun_out/r3y/m4_g20_dense.json 2> gpurun_out/r3y/m4_g20_dense.log
for f in gpurun_out/r3y/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; h=d['host_link']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), r.get('gather_kernels'), round(h.get('host_payload_GBps') or 0,1), round(d['stats']['feat_hit_rate'],3), d.get('parity_check',{}).get('bit_exact'), d['config']['position_table_MB_per_workspace'])" 2>&1 | tail -1; done
tail -2 gpurun_out/r3y/m4_g20_dense.log
