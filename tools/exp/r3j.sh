# session 3: L2 policy of the position tables in the sweeping hop (DCI_TABLE_POLICY 0 evict-last / 1 normal / 2 evict-first)
# and evict-first loads of the relabel's last use of candidates / counts (DCI_RELABEL_LASTUSE)
mkdir -p gpurun_out/r3j; rm -rf gpurun_out/r3j/*
DCI_TABLE_POLICY=0 DCI_RELABEL_LASTUSE=1 timeout 900 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py -q -x 2>&1 | tail -2 > gpurun_out/r3j/tests.txt
for i in 1 2; do
  for c in "1 0" "0 0" "2 0" "1 1" "0 1"; do
    set -- $c
    DCI_TABLE_POLICY=$1 DCI_RELABEL_LASTUSE=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3j/m2_$1$2_$i.json 2> /dev/null
  done
done
for c in "1 0" "0 0" "1 1"; do
  set -- $c
  DCI_TABLE_POLICY=$1 DCI_RELABEL_LASTUSE=$2 bash tools/exp/launches.sh tp$1$2 --steps 20 --warmup 5
done
cp gpurun_out/exp/launches_tp*.csv gpurun_out/r3j/
cat gpurun_out/r3j/tests.txt
for f in gpurun_out/r3j/*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(d['roofline']['frac'],3))"; done
