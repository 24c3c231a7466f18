mkdir -p gpurun_out/r2aa
timeout 900 ./tools/probe/vmm_host_probe 64 > gpurun_out/r2aa/vmm.jsonl 2> gpurun_out/r2aa/vmm.err
