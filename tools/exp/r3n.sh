# session 3: output-buffer allocation kind vs HBM write bandwidth (tools/probe/compress_probe.cu)
mkdir -p gpurun_out/r3n; rm -rf gpurun_out/r3n/*
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/compress_probe tools/probe/compress_probe.cu -lcuda
timeout 600 ./tools/probe/compress_probe > gpurun_out/r3n/compress_probe.jsonl 2> gpurun_out/r3n/compress_probe.err
for s in 0 10 20; do
  timeout 600 ncu --set full --clock-control none -k regex:k_wrand -s $s -c 1 -o gpurun_out/r3n/wrand_s$s ./tools/probe/compress_probe > /dev/null 2>&1
done
cat gpurun_out/r3n/compress_probe.jsonl gpurun_out/r3n/compress_probe.err
