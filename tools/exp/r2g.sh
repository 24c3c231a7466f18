# round-2 checks: full GPU tests, sanitizers over the group paths (incl. split gather), M2 bench as the driver runs it, M4 full size
mkdir -p gpurun_out/r2g gpurun_out/san
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r2g/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g/smoke.txt 2>&1
bash tools/sanitize.sh > gpurun_out/r2g/sanitize_summary.txt 2>&1
DCI_SPLIT_GATHER=1 timeout 600 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/smoke_racecheck_split.txt 2>&1
DCI_SPLIT_GATHER=1 timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/smoke_memcheck_split.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2g/bench_M2.json 2> gpurun_out/r2g/bench_M2.log
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2g/ref_M2.json 2> gpurun_out/r2g/ref_M2.log
free -g > gpurun_out/r2g/free.txt
timeout 2400 python bench.py --config M4 --steps 40 --warmup 8 --check-light --no-cpu-baseline > gpurun_out/r2g/bench_M4.json 2> gpurun_out/r2g/bench_M4.log
