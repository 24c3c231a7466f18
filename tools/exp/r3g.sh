# session 3: L2 policy of adjacency-cache element loads in the sampling hops (DCI_ELEM_POLICY 0 evict-last / 1 normal / 2 evict-first)
mkdir -p gpurun_out/r3g; rm -rf gpurun_out/r3g/*
for i in 1 2; do
  for p in 0 1 2; do
    DCI_ELEM_POLICY=$p timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3g/m2_p${p}_$i.json 2> gpurun_out/r3g/m2_p${p}_$i.log
  done
done
for p in 0 1 2; do DCI_ELEM_POLICY=$p bash tools/exp/launches.sh ep$p --steps 20 --warmup 5; done
cp gpurun_out/exp/launches_ep*.csv gpurun_out/r3g/
for f in gpurun_out/r3g/m2_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), round(d['roofline']['frac'],3))"; done
