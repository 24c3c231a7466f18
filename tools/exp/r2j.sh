# dynamic chunks in the sweep sampler; warp-parallel batch-table preambles
mkdir -p gpurun_out/r2j
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r2j/tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2j/bench_M2_k20.json 2> gpurun_out/r2j/bench_M2_k20.log
timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/r2j/bench_M2_k300.json 2> gpurun_out/r2j/bench_M2_k300.log
bash tools/exp/launches.sh r2j --steps 20 --warmup 5
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2j/bench_M1.json 2> gpurun_out/r2j/bench_M1.log
