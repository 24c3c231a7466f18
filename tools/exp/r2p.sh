# three-pass hop scan vs decoupled look-back
mkdir -p gpurun_out/r2p
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r2p/tests.txt
for sc in 3pass lookback; do
DCI_SCAN=$sc timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2p/bench_M2_k20_$sc.json 2> gpurun_out/r2p/bench_M2_k20_$sc.log
DCI_SCAN=$sc bash tools/exp/launches.sh r2p_$sc --steps 20 --warmup 5
done
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2p/bench_M1.json 2> gpurun_out/r2p/bench_M1.log
