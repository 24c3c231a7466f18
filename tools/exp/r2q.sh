mkdir -p gpurun_out/r2q
args="--profile-only --steps 20 --warmup 5 --repeats 1 --no-cpu-baseline"
ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:k_sample_hop -s 2 -c 1 -o gpurun_out/r2q/hop2 python bench.py $args > gpurun_out/r2q/hop2.stdout 2>&1
ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:k_sample_hop -s 1 -c 1 -o gpurun_out/r2q/hop1 python bench.py $args > gpurun_out/r2q/hop1.stdout 2>&1
