# session 3: confirm normal L2 policy for the sampler's element + directory loads (new default 1/1) vs the old evict-last (0/0)
mkdir -p gpurun_out/r3i; rm -rf gpurun_out/r3i/*
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r3i/gpu_tests.txt
for i in 1 2 3; do
  for c in "0 0" "1 1"; do
    set -- $c
    DCI_ELEM_POLICY=$1 DCI_DIR_POLICY=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3i/m2_$1$2_$i.json 2> /dev/null
  done
done
for i in 1 2; do
  for c in "0 0" "1 1"; do
    set -- $c
    DCI_ELEM_POLICY=$1 DCI_DIR_POLICY=$2 timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3i/m4s_$1$2_$i.json 2> /dev/null
  done
done
for c in "0 0" "1 1"; do
  set -- $c
  DCI_ELEM_POLICY=$1 DCI_DIR_POLICY=$2 timeout 900 python bench.py --config M1 --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3i/m1_$1$2.json 2> /dev/null
done
cat gpurun_out/r3i/gpu_tests.txt
for f in gpurun_out/r3i/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(d['roofline']['frac'],3))"; done
