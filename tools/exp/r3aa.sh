# session 3: groups of 20 + the host-aware sweep rule as the defaults (M3, M4s, M4), full GPU tests
mkdir -p gpurun_out/r3aa; rm -rf gpurun_out/r3aa/*
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r3aa/gpu_tests.txt
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 > gpurun_out/r3aa/bench_M3.json 2> gpurun_out/r3aa/bench_M3.log
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r3aa/bench_M4s.json 2> gpurun_out/r3aa/bench_M4s.log
timeout 2400 python bench.py --config M4 --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r3aa/bench_M4.json 2> gpurun_out/r3aa/bench_M4.log
cat gpurun_out/r3aa/gpu_tests.txt
for f in gpurun_out/r3aa/bench_*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; h=d['host_link']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), r.get('gather_kernels'), round(h.get('host_payload_GBps') or 0,1), round(d['stats']['feat_hit_rate'],3), d.get('parity_check',{}).get('bit_exact'), d['config']['position_table_MB_per_workspace'], d['config']['group'])" 2>&1 | tail -1; done
tail -2 gpurun_out/r3aa/bench_M4.log
