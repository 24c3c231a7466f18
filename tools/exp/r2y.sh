mkdir -p gpurun_out/r2y
timeout 900 ./tools/probe/hostreq_probe 64 m > gpurun_out/r2y/mixed.jsonl 2>&1
