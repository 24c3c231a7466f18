# session 3: L2 policies of the sampler's element (DCI_ELEM_POLICY) and directory (DCI_DIR_POLICY) loads on M2 / M3 / M4s
mkdir -p gpurun_out/r3h; rm -rf gpurun_out/r3h/*
for i in 1 2; do
  for c in "0 0" "2 0" "2 1" "2 2" "1 1"; do
    set -- $c
    DCI_ELEM_POLICY=$1 DCI_DIR_POLICY=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3h/m2_$1$2_$i.json 2> /dev/null
  done
done
for c in "0 0" "2 0" "2 1" "1 1"; do
  set -- $c
  DCI_ELEM_POLICY=$1 DCI_DIR_POLICY=$2 timeout 900 python bench.py --config M3 --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3h/m3_$1$2.json 2> /dev/null
  DCI_ELEM_POLICY=$1 DCI_DIR_POLICY=$2 timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3h/m4s_$1$2.json 2> /dev/null
done
for f in gpurun_out/r3h/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(d['roofline']['frac'],3))"; done
