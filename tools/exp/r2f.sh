mkdir -p gpurun_out/r2f
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2f/tests.txt
for sp in 1 0; do
DCI_SPLIT_GATHER=$sp timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2f/bench_M2_k20_split$sp.json 2> gpurun_out/r2f/bench_M2_k20_split$sp.log
done
timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/r2f/bench_M2_k300.json 2> gpurun_out/r2f/bench_M2_k300.log
bash tools/exp/launches.sh r2f --steps 20 --warmup 5
timeout 900 ./tools/probe/hostreq_probe 64 > gpurun_out/r2f/hostreq.jsonl 2>&1
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2f/bench_M3.json 2> gpurun_out/r2f/bench_M3.log
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline > gpurun_out/r2f/bench_M4s.json 2> gpurun_out/r2f/bench_M4s.log
