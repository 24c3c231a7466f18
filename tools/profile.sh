#!/bin/bash
# ncu evidence for the hot path (run under gpurun; 1 GPU).  Usage: tools/profile.sh <tag> [bench args...]
# Only kernels inside bench.py's NVTX range "timed" are profiled.
tag=${1:-run}; shift
out=gpurun_out/prof_$tag; mkdir -p $out
args="--profile-only --steps 40 --warmup 20 --repeats 1 --no-cpu-baseline $@"
nv="--nvtx --nvtx-include timed/"
ncu $nv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py $args > $out/launches.stdout 2>&1
ncu $nv --set full --clock-control none --import-source on -k regex:k_gather -s 1 -c 2 -o $out/gather \
    python bench.py $args > $out/gather.stdout 2>&1
ncu $nv --set full --clock-control none --import-source on -k regex:k_sample_hop -s 3 -c 3 -o $out/sample \
    python bench.py $args > $out/sample.stdout 2>&1
ncu $nv --set full --clock-control none --import-source on -k regex:"k_scan_hop" -s 3 -c 3 -o $out/scan \
    python bench.py $args > $out/scan.stdout 2>&1
ls -la $out
