timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/final_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/final_tests.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_M2.json 2> gpurun_out/bench_M2.log
timeout 600 python bench.py --config M1 > gpurun_out/bench_M1.json 2> gpurun_out/bench_M1.log
timeout 900 python bench.py --config M3 > gpurun_out/bench_M3.json 2> gpurun_out/bench_M3.log
timeout 600 python bench.py --impl reference > gpurun_out/ref_M2.json 2> gpurun_out/ref_M2.log
bash tools/profile.sh r01z > /dev/null 2>&1
cat gpurun_out/final_tests.txt
python -c "
import json
for c in ['M2','M1','M3']:
    d=json.load(open('gpurun_out/bench_%s.json'%c)); r=d['roofline']
    print(c, d['steps'], d['value'], d['e2e']['value'], r['frac'], (r.get('pattern') or {}).get('frac'), d.get('parity_check',{}).get('bit_exact'), d.get('cpu_baseline',{}).get('value'), d['clocks']['reasons'])"
