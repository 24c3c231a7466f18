# session 3 final check of HEAD: GPU tests, smoke, the driver's bench command, reference arm, launch list
mkdir -p gpurun_out/fin4; rm -rf gpurun_out/fin4/*
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/fin4/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4/smoke.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin4/bench_M2_k20.json 2> gpurun_out/fin4/bench_M2_k20.log
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin4/reference_M2.json 2> gpurun_out/fin4/reference_M2.log
bash tools/exp/launches.sh fin4 --steps 20 --warmup 5; cp gpurun_out/exp/launches_fin4.csv gpurun_out/fin4/launches_m2.csv
cat gpurun_out/fin4/gpu_tests.txt gpurun_out/fin4/smoke.txt
python -c "
import json; d=json.load(open('gpurun_out/fin4/bench_M2_k20.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'], d['parity_check'], d['clocks']['reasons'], d['cpu_baseline']['value'])"
