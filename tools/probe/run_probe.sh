#!/bin/bash
# Box probe: topology, host, host-link microbenchmarks. Output under gpurun_out/probe/.
mkdir -p gpurun_out/probe
nvidia-smi -q > gpurun_out/probe/nvsmi_q.txt 2>&1
nvidia-smi topo -m > gpurun_out/probe/topo.txt 2>&1
(free -g; nproc; lscpu; ulimit -l; cat /proc/meminfo | head -5) > gpurun_out/probe/host.txt 2>&1
nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv >> gpurun_out/probe/host.txt 2>&1
timeout 300 ./tools/probe/hostlink_probe > gpurun_out/probe/probe.jsonl 2>&1
echo "probe exit $?" >> gpurun_out/probe/probe.jsonl
