mkdir -p gpurun_out/r2mm
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 > gpurun_out/r2mm/bench_M3.json 2> gpurun_out/r2mm/bench_M3.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2mm/bench_M2_k20.json 2> gpurun_out/r2mm/bench_M2_k20.log
