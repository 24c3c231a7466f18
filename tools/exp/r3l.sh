# session 3: scan tickets interleaved over the batches of a group (DCI_SCAN_INTERLEAVE) -- parity + A/B
mkdir -p gpurun_out/r3l; rm -rf gpurun_out/r3l/*
DCI_SCAN_INTERLEAVE=1 timeout 1200 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 > gpurun_out/r3l/tests.txt
for i in 1 2 3; do
  for c in 0 1; do
    DCI_SCAN_INTERLEAVE=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3l/m2_${c}_$i.json 2> /dev/null
  done
done
for c in 0 1; do DCI_SCAN_INTERLEAVE=$c bash tools/exp/launches.sh si$c --steps 20 --warmup 5; done
cp gpurun_out/exp/launches_si*.csv gpurun_out/r3l/
cat gpurun_out/r3l/tests.txt
for f in gpurun_out/r3l/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(d['roofline']['frac'],3))"; done
