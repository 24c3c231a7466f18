mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --target-processes all python -m pytest tests/test_gpu_many.py -q -x -k "not stats" > gpurun_out/san/many_$t.txt 2>&1
  tail -3 gpurun_out/san/many_$t.txt
done
timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/smoke_memcheck.txt 2>&1; tail -2 gpurun_out/san/smoke_memcheck.txt
