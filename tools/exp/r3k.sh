# session 3: which hops sample by node sweep (DCI_SWEEP_FACTOR: a hop sweeps when its frontier total >= factor x N)
mkdir -p gpurun_out/r3k; rm -rf gpurun_out/r3k/*
DCI_SWEEP_FACTOR=2 timeout 900 python -m pytest tests/test_gpu_many.py -q -x 2>&1 | tail -2 > gpurun_out/r3k/tests.txt
for i in 1 2; do
  for fct in 1 2 0.5; do
    DCI_SWEEP_FACTOR=$fct timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3k/m2_f${fct}_$i.json 2> /dev/null
  done
done
for fct in 1 2; do DCI_SWEEP_FACTOR=$fct bash tools/exp/launches.sh sf$fct --steps 20 --warmup 5; done
cp gpurun_out/exp/launches_sf*.csv gpurun_out/r3k/
cat gpurun_out/r3k/tests.txt
for f in gpurun_out/r3k/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(d['roofline']['frac'],3))"; done
