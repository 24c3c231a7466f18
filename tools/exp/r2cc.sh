mkdir -p gpurun_out/r2cc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cc/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r2cc/tests.txt
DCI_SAMPLE_SWEEP=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cc/smoke_nosweep.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cc/smoke_memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cc/smoke_racecheck.txt 2>&1
