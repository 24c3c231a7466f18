# session 3 final closing run with every default in place: tests, smoke, bench lines M1-M4 + reference, launch list
mkdir -p gpurun_out/fin5; rm -rf gpurun_out/fin5/*
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/fin5/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin5/smoke.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin5/bench_M2_k20.json 2> gpurun_out/fin5/bench_M2_k20.log
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin5/reference_M2.json 2> gpurun_out/fin5/reference_M2.log
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 > gpurun_out/fin5/bench_M1.json 2> gpurun_out/fin5/bench_M1.log
timeout 900 python bench.py --config M3 --steps 64 --warmup 8 > gpurun_out/fin5/bench_M3.json 2> gpurun_out/fin5/bench_M3.log
timeout 900 python bench.py --config M4s --steps 64 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/fin5/bench_M4s.json 2> gpurun_out/fin5/bench_M4s.log
timeout 2400 python bench.py --config M4 --steps 64 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/fin5/bench_M4.json 2> gpurun_out/fin5/bench_M4.log
bash tools/exp/launches.sh fin5 --steps 20 --warmup 5; cp gpurun_out/exp/launches_fin5.csv gpurun_out/fin5/launches_m2.csv
cat gpurun_out/fin5/gpu_tests.txt gpurun_out/fin5/smoke.txt
for f in gpurun_out/fin5/bench_*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; s=d['stats']; print('$f', d['steps'], round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['frac'] or 0,3), d.get('parity_check',{}).get('bit_exact'), (d.get('cpu_baseline') or {}).get('value'), d['clocks']['reasons'], s.get('eq1_times'))" 2>&1 | tail -1; done
