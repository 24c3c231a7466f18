#!/bin/bash
# ncu host-link evidence for host-link-bound configs (PCIe read bytes / throughput, sysmem requests).
# Usage: tools/profile_hostlink.sh <tag> <bench args...>   (run under gpurun; 1 GPU)
tag=$1; shift
out=gpurun_out/prof_hl_$tag; mkdir -p $out
ncu --nvtx --nvtx-include timed/ --clock-control none -k regex:"k_gather|k_sample_hop" -s 4 -c 8 \
    --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed,syslts__t_requests_aperture_sysmem.sum,syslts__d_sectors_fill_sysmem.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --csv --log-file $out/hostlink.csv python bench.py --profile-only --steps 6 --warmup 2 --no-cpu-baseline --inflight 1 "$@" > $out/stdout 2>&1
ls -la $out
