# session 3: row-layout relabel (DCI_RELABEL_ROWS) -- parity + A/B at K=20
mkdir -p gpurun_out/r3e; rm -rf gpurun_out/r3e/*
timeout 1500 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3 > gpurun_out/r3e/tests.txt
for i in 1 2 3; do
  for c in 0 1; do
    DCI_RELABEL_ROWS=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3e/m2_${c}_$i.json 2> gpurun_out/r3e/m2_${c}_$i.log
  done
done
for c in 0 1; do DCI_RELABEL_ROWS=$c bash tools/exp/launches.sh rr$c --steps 20 --warmup 5; done
cp gpurun_out/exp/launches_rr*.csv gpurun_out/r3e/
cat gpurun_out/r3e/tests.txt
for f in gpurun_out/r3e/m2_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), round(d['roofline']['frac'],3), round(d['roofline']['avg_gather_ms'],4))"; done
