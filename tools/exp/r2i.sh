mkdir -p gpurun_out/r2i
args="--profile-only --steps 20 --warmup 5 --repeats 1 --no-cpu-baseline"
ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:k_sample_hop -s 2 -c 1 -o gpurun_out/r2i/hop2 python bench.py $args > gpurun_out/r2i/hop2.stdout 2>&1
ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:"k_scan_hop|k_newmask" -s 4 -c 2 -o gpurun_out/r2i/scan2 python bench.py $args > gpurun_out/r2i/scan2.stdout 2>&1
ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:k_hop_epilogue -c 1 -o gpurun_out/r2i/epi python bench.py $args > gpurun_out/r2i/epi.stdout 2>&1
