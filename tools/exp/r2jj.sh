mkdir -p gpurun_out/r2jj
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/r2jj/tests.txt
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2jj/pdl$i.json 2> gpurun_out/r2jj/pdl$i.log
DCI_PDL=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2jj/nopdl$i.json 2> gpurun_out/r2jj/nopdl$i.log
done
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2jj/M1_pdl.json 2> gpurun_out/r2jj/M1_pdl.log
DCI_PDL=0 timeout 600 python bench.py --config M1 --steps 20 --warmup 5 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2jj/M1_nopdl.json 2> gpurun_out/r2jj/M1_nopdl.log
timeout 900 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2jj/smoke_racecheck.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2jj/smoke_synccheck.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2jj/smoke_memcheck.txt 2>&1
