# session 3: scan preloads a sweeping hop's new candidates (DCI_SCAN_PREX) -- parity + A/B at K=20
mkdir -p gpurun_out/r3b; rm -rf gpurun_out/r3b/*
timeout 1200 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3 > gpurun_out/r3b/tests.txt
for i in 1 2; do
  for p in 0 1; do
    DCI_SCAN_PREX=$p timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3b/m2_p${p}_$i.json 2> gpurun_out/r3b/m2_p${p}_$i.log
  done
done
DCI_SCAN_PREX=0 bash tools/exp/launches.sh p0 --steps 20 --warmup 5
DCI_SCAN_PREX=1 bash tools/exp/launches.sh p1 --steps 20 --warmup 5
cp gpurun_out/exp/launches_p*.csv gpurun_out/r3b/
cat gpurun_out/r3b/tests.txt
for f in gpurun_out/r3b/m2_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), round(d['roofline']['frac'],3), d.get('parity_check',{}).get('bit_exact'))"; done
