# ncu DRAM counters of the scatter probe's kernels (the sweep gather's write pattern), P = 2432
mkdir -p gpurun_out/r2bb
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/r2bb/scatter_ncu.csv ./tools/probe/scatter_probe 232965 2432 141187 20 > gpurun_out/r2bb/scatter.stdout 2>&1
