#!/bin/bash
# ncu --set full of one node-sweep gather launch (M2, group of 20) -> gpurun_out/exp/sweep.ncu-rep
mkdir -p gpurun_out/exp
ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:k_gather_sweep -s 1 -c 1 \
  -o gpurun_out/exp/sweep python bench.py --profile-only --steps 40 --warmup 20 --repeats 1 --no-cpu-baseline $@ \
  > gpurun_out/exp/sweep_ncu.stdout 2>&1
ncu -i gpurun_out/exp/sweep.ncu-rep --page raw --csv > gpurun_out/exp/sweep_raw.csv 2>&1
ncu -i gpurun_out/exp/sweep.ncu-rep --page source --csv > gpurun_out/exp/sweep_source.csv 2>&1
