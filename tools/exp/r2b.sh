# round 2: ncu evidence for the current default (M2) + host-link configs + bench lines
mkdir -p gpurun_out/r2b
bash tools/profile.sh r02 > /dev/null 2>&1
bash tools/profile_hostlink.sh m3 --config M3 > /dev/null 2>&1
bash tools/profile_hostlink.sh m4s --config M4s --group 8 --inflight 1 > /dev/null 2>&1
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 > gpurun_out/r2b/bench_M1.json 2> gpurun_out/r2b/bench_M1.log
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 > gpurun_out/r2b/bench_M3.json 2> gpurun_out/r2b/bench_M3.log
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r2b/bench_M4s.json 2> gpurun_out/r2b/bench_M4s.log
