# session 3: final lines of the host-resident configs under the new defaults (groups of 20, node sweeps), and M2
mkdir -p gpurun_out/r3bb; rm -rf gpurun_out/r3bb/*
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 > gpurun_out/r3bb/bench_M3.json 2> gpurun_out/r3bb/bench_M3.log
timeout 900 python bench.py --config M3 --steps 100 --warmup 20 --no-cpu-baseline > gpurun_out/r3bb/bench_M3_k100.json 2> gpurun_out/r3bb/bench_M3_k100.log
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r3bb/bench_M4s.json 2> gpurun_out/r3bb/bench_M4s.log
timeout 2400 python bench.py --config M4 --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r3bb/bench_M4.json 2> gpurun_out/r3bb/bench_M4.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r3bb/bench_M2_k20.json 2> gpurun_out/r3bb/bench_M2_k20.log
bash tools/profile_hostlink.sh m4s_sweep --config M4s > /dev/null 2>&1; cp gpurun_out/prof_hl_m4s_sweep/hostlink.csv gpurun_out/r3bb/hostlink_m4s_sweep.csv
for f in gpurun_out/r3bb/bench_*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; h=d['host_link']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['frac'],3), r['peak'], round(h.get('host_payload_GBps') or 0,1), (h.get('step_roofline') or {}).get('frac'), d.get('parity_check',{}).get('bit_exact'))" 2>&1 | tail -1; done
