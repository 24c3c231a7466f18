#!/bin/bash
# ncu launch list (per-launch time + DRAM bytes) of the bench's timed region -> gpurun_out/exp/launches_<tag>.csv
tag=${1:-m2}; shift
mkdir -p gpurun_out/exp
ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/exp/launches_$tag.csv \
  python bench.py --profile-only --repeats 1 --no-cpu-baseline "$@" > gpurun_out/exp/launches_$tag.stdout 2>&1
