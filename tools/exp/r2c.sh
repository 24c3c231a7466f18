# probes: host-link request rate by region/size; HBM scatter pattern (P=2432 line rows, 2416 pitch rows); ncu of the TMA sweep gather
mkdir -p gpurun_out/r2c
timeout 300 ./tools/probe/scatter_probe 232965 2432 141187 20 > gpurun_out/r2c/scatter_2432.jsonl 2>&1
timeout 300 ./tools/probe/scatter_probe 232965 2416 141187 20 > gpurun_out/r2c/scatter_2416.jsonl 2>&1
timeout 600 ./tools/probe/hostreq_probe 64 > gpurun_out/r2c/hostreq.jsonl 2>&1
ncu --nvtx --nvtx-include timed/ --set full --clock-control none --import-source on -k regex:k_gather_sweep_tma -c 1 -o gpurun_out/r2c/gather_sweep_tma \
    python bench.py --profile-only --steps 20 --warmup 5 --repeats 1 --no-cpu-baseline > gpurun_out/r2c/gather_sweep_tma.stdout 2>&1
