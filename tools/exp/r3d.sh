# session 3: L1-allocating tag loads -- precheck before the atomicMax (DCI_PRECHECK=2) and the relabel (DCI_RELABEL_L1=1)
mkdir -p gpurun_out/r3d; rm -rf gpurun_out/r3d/*
DCI_PRECHECK=2 DCI_RELABEL_L1=1 timeout 1200 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py -q -x 2>&1 | tail -3 > gpurun_out/r3d/tests.txt
for i in 1 2; do
  for c in "0 0" "2 0" "0 1" "2 1"; do
    set -- $c
    DCI_PRECHECK=$1 DCI_RELABEL_L1=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3d/m2_$1$2_$i.json 2> gpurun_out/r3d/m2_$1$2_$i.log
  done
done
for c in "0 0" "2 0" "0 1" "2 1"; do
  set -- $c
  DCI_PRECHECK=$1 DCI_RELABEL_L1=$2 bash tools/exp/launches.sh c$1$2 --steps 20 --warmup 5
done
cp gpurun_out/exp/launches_c*.csv gpurun_out/r3d/
cat gpurun_out/r3d/tests.txt
for f in gpurun_out/r3d/m2_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), round(d['roofline']['frac'],3), d.get('parity_check',{}).get('bit_exact'))"; done
