# session 3: ncu PCIe / sysmem counters of the host-resident configs under the final defaults (node-sweep groups)
mkdir -p gpurun_out/r3gg; rm -rf gpurun_out/r3gg/*
bash tools/profile_hostlink.sh m3_final --config M3 > /dev/null 2>&1; cp gpurun_out/prof_hl_m3_final/hostlink.csv gpurun_out/r3gg/hostlink_m3.csv
bash tools/profile_hostlink.sh m4s_final --config M4s > /dev/null 2>&1; cp gpurun_out/prof_hl_m4s_final/hostlink.csv gpurun_out/r3gg/hostlink_m4s.csv
ls -la gpurun_out/r3gg
