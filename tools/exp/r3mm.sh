# session 3: a lower sampling-sweep threshold (DCI_SWEEP_FACTOR=0.015: M4's last hop and M3's hop 1 sweep too)
mkdir -p gpurun_out/r3mm; rm -rf gpurun_out/r3mm/*
for fct in 0.05 0.015; do
  DCI_SWEEP_FACTOR=$fct timeout 900 python bench.py --config M3 --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3mm/m3_f$fct.json 2> /dev/null
  DCI_SWEEP_FACTOR=$fct timeout 900 python bench.py --config M4s --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3mm/m4s_f$fct.json 2> /dev/null
  DCI_SWEEP_FACTOR=$fct timeout 2400 python bench.py --config M4 --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3mm/m4_f$fct.json 2> /dev/null
done
for f in gpurun_out/r3mm/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['avg_sample_ms'],3), round(r['avg_gather_ms'],2))"; done
