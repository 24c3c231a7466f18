# session 3 closing evidence with the final code (one B200): tests, smoke, sanitizers, bench lines M1-M4 + reference, ncu
mkdir -p gpurun_out/fin3 gpurun_out/san; rm -rf gpurun_out/fin3/* gpurun_out/prof_fin3 gpurun_out/san/*
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/fin3/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3/smoke.txt 2>&1
bash tools/sanitize.sh > gpurun_out/fin3/sanitize_summary.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin3/bench_M2_k20.json 2> gpurun_out/fin3/bench_M2_k20.log
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin3/reference_M2.json 2> gpurun_out/fin3/reference_M2.log
timeout 600 python bench.py --gpus 1 --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/fin3/bench_M2_k300.json 2> gpurun_out/fin3/bench_M2_k300.log
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 > gpurun_out/fin3/bench_M1.json 2> gpurun_out/fin3/bench_M1.log
timeout 900 python bench.py --config M3 --steps 20 --warmup 5 > gpurun_out/fin3/bench_M3.json 2> gpurun_out/fin3/bench_M3.log
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/fin3/bench_M4s.json 2> gpurun_out/fin3/bench_M4s.log
bash tools/profile.sh fin3 > /dev/null 2>&1
ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:k_gather_sweep_tma -c 1 -o gpurun_out/fin3/gather_sweep_tma python bench.py --profile-only --steps 20 --warmup 5 --repeats 1 --no-cpu-baseline > gpurun_out/fin3/gst.stdout 2>&1
bash tools/profile_hostlink.sh m3 --config M3 > /dev/null 2>&1
bash tools/profile_hostlink.sh m4s --config M4s --group 8 --inflight 1 > /dev/null 2>&1
timeout 2400 python bench.py --config M4 --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/fin3/bench_M4.json 2> gpurun_out/fin3/bench_M4.log
cp -r gpurun_out/san gpurun_out/fin3/sanitizer; cp -r gpurun_out/prof_hl_m3 gpurun_out/prof_hl_m4s gpurun_out/fin3/ 2>/dev/null; cat gpurun_out/fin3/gpu_tests.txt gpurun_out/fin3/smoke.txt
