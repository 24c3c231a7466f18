#!/bin/bash
# SURVEY §7 step 0 / §8(e) caveat: N GPUs reading ONE pinned host region at once (1, 2, 4, 8 readers,
# as many as are visible).  Builds the probe and writes profiles/hostlink_<n>reader.json, n = the
# visible device count.  Usage: tools/probe/run_multireader.sh [region_GB=8]
set -e
cd "$(dirname "$0")/../.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/multireader_probe tools/probe/multireader_probe.cu
n=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out/probe
timeout 900 ./tools/probe/multireader_probe "${1:-8}" gpurun_out/probe/hostlink_${n}reader.json
cp gpurun_out/probe/hostlink_${n}reader.json profiles/hostlink_${n}reader.json 2>/dev/null || true
