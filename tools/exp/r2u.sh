mkdir -p gpurun_out/r2u
timeout 1200 ./tools/probe/hostreq_probe 64 > gpurun_out/r2u/hostreq.jsonl 2>&1
