# session 3: scan tiles of 128 dsts (kScanTile = 128, built into libdci_t128.so) vs 256
mkdir -p gpurun_out/r3u; rm -rf gpurun_out/r3u/*
V=$PWD/paper_2503_01281_b200/libdci_t128.so
DCI_LIB=$V timeout 1200 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py -q -x 2>&1 | tail -2 > gpurun_out/r3u/tests.txt
for i in 1 2 3; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3u/m2_256_$i.json 2> /dev/null
  DCI_LIB=$V timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency --no-aggregate > gpurun_out/r3u/m2_128_$i.json 2> /dev/null
done
bash tools/exp/launches.sh t256 --steps 20 --warmup 5
DCI_LIB=$V bash tools/exp/launches.sh t128 --steps 20 --warmup 5
cp gpurun_out/exp/launches_t*.csv gpurun_out/r3u/
cat gpurun_out/r3u/tests.txt
for f in gpurun_out/r3u/m2_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['value']/1e6,4), round(d['e2e']['value']/1e6,4))"; done
