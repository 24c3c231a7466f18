# session 3: L2 prefetch size of the sampler's host adjacency reads (DCI_HOST_PREFETCH 0 / 64 / 128 / 256 B)
mkdir -p gpurun_out/r3ee; rm -rf gpurun_out/r3ee/*
DCI_HOST_PREFETCH=2 timeout 900 python -m pytest tests/test_gpu_random.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > gpurun_out/r3ee/tests.txt
for p in 0 1 2 3; do
  DCI_HOST_PREFETCH=$p timeout 900 python bench.py --config M3 --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ee/m3_p$p.json 2> /dev/null
  DCI_HOST_PREFETCH=$p timeout 900 python bench.py --config M4s --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ee/m4s_p$p.json 2> /dev/null
done
for p in 0 2 3; do
  DCI_HOST_PREFETCH=$p timeout 2400 python bench.py --config M4 --steps 64 --warmup 8 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3ee/m4_p$p.json 2> /dev/null
done
cat gpurun_out/r3ee/tests.txt
for f in gpurun_out/r3ee/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4), round(r['avg_sample_ms'],3), round(r['avg_gather_ms'],2))"; done
