mkdir -p gpurun_out/r2e
timeout 600 ./tools/probe/hostreq_probe 8 > gpurun_out/r2e/hostreq.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2e/tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e/bench_M2_k20.json 2> gpurun_out/r2e/bench_M2_k20.log
timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/r2e/bench_M2_k300.json 2> gpurun_out/r2e/bench_M2_k300.log
bash tools/exp/launches.sh r2e --steps 20 --warmup 5
