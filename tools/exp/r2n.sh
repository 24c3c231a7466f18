# sweep sampler: block ranges + shared tickets, tag bases, nmask zeroing pass
mkdir -p gpurun_out/r2n
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r2n/tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2n/bench_M2_k20.json 2> gpurun_out/r2n/bench_M2_k20.log
bash tools/exp/launches.sh r2n --steps 20 --warmup 5
timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/r2n/bench_M2_k300.json 2> gpurun_out/r2n/bench_M2_k300.log
