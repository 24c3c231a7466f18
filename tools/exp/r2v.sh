# adjacency-miss runs counted; host-link request view
mkdir -p gpurun_out/r2v
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r2v/tests.txt
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2v/bench_M3.json 2> gpurun_out/r2v/bench_M3.log
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --no-check > gpurun_out/r2v/bench_M4s.json 2> gpurun_out/r2v/bench_M4s.log
timeout 2400 python bench.py --config M4 --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r2v/bench_M4.json 2> gpurun_out/r2v/bench_M4.log
