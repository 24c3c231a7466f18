# M4s/M4: is the group gather's host-row rate bound by the region (TLB) or by the sampler beside it?
mkdir -p gpurun_out/r2r
for ph in 0 1; do
DCI_PHASED=$ph timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --no-check > gpurun_out/r2r/M4s_ph$ph.json 2> gpurun_out/r2r/M4s_ph$ph.log
done
for n in 8 64; do
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --no-cpu-baseline --no-check --presample-batches $n > gpurun_out/r2r/M4s_pre$n.json 2> gpurun_out/r2r/M4s_pre$n.log
done
