# sweep-sampler chunk size: 0 (static stride), 4, 16, 64 node groups per ticket
mkdir -p gpurun_out/r2k
for c in 0 16 64 4; do
DCI_SAMPLE_CHUNK=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-check > gpurun_out/r2k/bench_c$c.json 2> gpurun_out/r2k/bench_c$c.log
DCI_SAMPLE_CHUNK=$c bash tools/exp/launches.sh r2k_c$c --steps 20 --warmup 5
done
