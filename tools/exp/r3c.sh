# session 3: source-level ncu captures of the last hop, its scan and the relabel epilogue (M2, K=20)
mkdir -p gpurun_out/r3c; rm -rf gpurun_out/r3c/*
args="--profile-only --steps 20 --warmup 5 --repeats 1 --no-cpu-baseline"
nv="--nvtx --nvtx-include timed/"
ncu $nv --set full --clock-control none --import-source on -k regex:k_sample_hop -s 2 -c 1 -o gpurun_out/r3c/hop2 python bench.py $args > gpurun_out/r3c/hop2.stdout 2>&1
ncu $nv --set full --clock-control none --import-source on -k regex:k_scan_hop -s 2 -c 1 -o gpurun_out/r3c/scan2 python bench.py $args > gpurun_out/r3c/scan2.stdout 2>&1
ncu $nv --set full --clock-control none --import-source on -k regex:k_hop_epilogue -c 1 -o gpurun_out/r3c/epi python bench.py $args > gpurun_out/r3c/epi.stdout 2>&1
ls -la gpurun_out/r3c
