# session 3: final lines of the host-resident configs with groups of 32 (K = 64: two full groups)
mkdir -p gpurun_out/r3dd; rm -rf gpurun_out/r3dd/*
timeout 900 python bench.py --config M3 --steps 64 --warmup 8 > gpurun_out/r3dd/bench_M3.json 2> gpurun_out/r3dd/bench_M3.log
timeout 900 python bench.py --config M4s --steps 64 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r3dd/bench_M4s.json 2> gpurun_out/r3dd/bench_M4s.log
timeout 2400 python bench.py --config M4 --steps 64 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r3dd/bench_M4.json 2> gpurun_out/r3dd/bench_M4.log
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3dd/bench_M3_k20.json 2> /dev/null
for f in gpurun_out/r3dd/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; h=d['host_link']; print('$f', d['steps'], d['config']['group'], round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['frac'],3), round(h.get('host_payload_GBps') or 0,1), round((h.get('step_roofline') or {}).get('frac') or 0,3), d.get('parity_check',{}).get('bit_exact'), (d.get('cpu_baseline') or {}).get('value'))" 2>&1 | tail -1; done
