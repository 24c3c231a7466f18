# session-3 re-entry check of HEAD (one B200): GPU tests, smoke, driver-style M2 bench
mkdir -p gpurun_out/r3a; rm -rf gpurun_out/r3a/*
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r3a/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r3a/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r3a/smoke.txt
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r3a/bench_M2_k20.json 2> gpurun_out/r3a/bench_M2_k20.log
cat gpurun_out/r3a/gpu_tests.txt gpurun_out/r3a/smoke.txt
python -c "
import json; d=json.load(open('gpurun_out/r3a/bench_M2_k20.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
