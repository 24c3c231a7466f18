# session 3: M1 (10 K nodes, latency-bound) with the node-sweep gather / sampling vs row mode
mkdir -p gpurun_out/r3w; rm -rf gpurun_out/r3w/*
for i in 1 2; do
  for c in "1 1" "0 1" "0 0" "1 0"; do
    set -- $c
    DCI_SWEEP=$1 DCI_SAMPLE_SWEEP=$2 timeout 600 python bench.py --config M1 --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3w/m1_$1$2_$i.json 2> /dev/null
  done
done
DCI_SWEEP=0 bash tools/exp/launches.sh m1s0 --config M1 --steps 20 --warmup 5; cp gpurun_out/exp/launches_m1s0.csv gpurun_out/r3w/
for f in gpurun_out/r3w/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3))"; done
