# node-major new-candidate masks for sweeping hops; group size at the driver's K=20
mkdir -p gpurun_out/r2h
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r2h/tests.txt
for g in 20 10; do
timeout 600 python bench.py --steps 20 --warmup 5 --group $g --no-cpu-baseline > gpurun_out/r2h/bench_M2_k20_g$g.json 2> gpurun_out/r2h/bench_M2_k20_g$g.log
done
DCI_NMASK_SWEEP=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2h/bench_M2_k20_nonmask.json 2> gpurun_out/r2h/bench_M2_k20_nonmask.log
timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/r2h/bench_M2_k300.json 2> gpurun_out/r2h/bench_M2_k300.log
bash tools/exp/launches.sh r2h --steps 20 --warmup 5
for g in 8 0; do
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --group $g --no-cpu-baseline > gpurun_out/r2h/bench_M4s_g$g.json 2> gpurun_out/r2h/bench_M4s_g$g.log
done
