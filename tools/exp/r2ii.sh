mkdir -p gpurun_out/r2ii
timeout 900 python -m pytest tests/test_gpu_many.py tests/test_gpu_random.py -q -x 2>&1 | tail -3 > gpurun_out/r2ii/tests.txt
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2ii/b$i.json 2> gpurun_out/r2ii/b$i.log; done
bash tools/exp/launches.sh r2ii --steps 20 --warmup 5
