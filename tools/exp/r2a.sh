mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r2a/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2a/bench_M2.json 2> gpurun_out/r2a/bench_M2.log
timeout 600 python bench.py --gpus 1 --steps 300 --warmup 20 > gpurun_out/r2a/bench_M2_k300.json 2> gpurun_out/r2a/bench_M2_k300.log
bash tools/exp/launches.sh m2 --steps 20 --warmup 5
