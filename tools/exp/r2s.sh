# F3 presample-count sweep on papers100M-shaped graphs (Fig. 11 analogue beyond products)
mkdir -p gpurun_out/r2s
for n in 8 16 32 64 128 256; do
timeout 900 python bench.py --config M4s --steps 40 --warmup 8 --repeats 3 --no-cpu-baseline --no-check --presample-batches $n > gpurun_out/r2s/M4s_pre$n.json 2> gpurun_out/r2s/M4s_pre$n.log
done
for n in 64 256; do
timeout 2400 python bench.py --config M4 --steps 40 --warmup 8 --repeats 3 --no-cpu-baseline --no-check --presample-batches $n > gpurun_out/r2s/M4_pre$n.json 2> gpurun_out/r2s/M4_pre$n.log
done
