# scan: warp-cooperative new-node append, binary-searched tile -> batch
mkdir -p gpurun_out/r2o
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r2o/tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2o/bench_M2_k20.json 2> gpurun_out/r2o/bench_M2_k20.log
bash tools/exp/launches.sh r2o --steps 20 --warmup 5
