# TMA gather: GPU tests, then a parameter sweep on M2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/exp2_tests.txt
S=gpurun_out/exp2_sweep.txt
DCI_GATHER=ldg bash tools/sweep.sh "ldg" --inflight 6 --steps 300 --no-check >> $S 2>&1
for cfg in "tma_w4_200_8k:" "tma_w2_200_8k:DCI_TMA_WARPS=2" "tma_w8_200_8k:DCI_TMA_WARPS=8" "tma_w4_100_8k:DCI_TMA_SMEM_KB=100" "tma_w4_200_4k:DCI_TMA_CHUNK=4096" "tma_w4_200_16k:DCI_TMA_CHUNK=16384" "tma_w4_150_8k:DCI_TMA_SMEM_KB=150"; do
  lab=${cfg%%:*}; envs=${cfg#*:}
  for inf in 4 8; do
    env $envs bash tools/sweep.sh "$lab" --inflight $inf --steps 300 --no-check >> $S 2>&1
  done
done
cat gpurun_out/exp2_tests.txt $S
