# session 3: node-sweep TMA gather storing from registers (DCI_SWEEP_REGSTORE=1) instead of bulk shared->global copies
mkdir -p gpurun_out/r3p; rm -rf gpurun_out/r3p/*
DCI_SWEEP_REGSTORE=1 timeout 1200 python -m pytest tests/test_gpu_many.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 > gpurun_out/r3p/tests.txt
for i in 1 2 3; do
  for c in 0 1; do
    DCI_SWEEP_REGSTORE=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3p/m2_${c}_$i.json 2> /dev/null
  done
done
for c in 0 1; do DCI_SWEEP_REGSTORE=$c bash tools/exp/launches.sh rs$c --steps 20 --warmup 5; done
cp gpurun_out/exp/launches_rs*.csv gpurun_out/r3p/
cat gpurun_out/r3p/tests.txt
for f in gpurun_out/r3p/*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['frac'],3), round(r['avg_gather_ms'],4), (r.get('alone') or {}).get('avg_gather_ms'))"; done
