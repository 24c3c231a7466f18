S=gpurun_out/exp3_sweep.txt
for inf in 1 2; do
  DCI_GATHER=ldg bash tools/sweep.sh "ldg" --inflight $inf --steps 200 --no-check >> $S 2>&1
  bash tools/sweep.sh "tma" --inflight $inf --steps 200 --no-check >> $S 2>&1
done
for inf in 4 6 8; do
  DCI_GATHER_SERIAL=0 bash tools/sweep.sh "tma_conc" --inflight $inf --steps 300 --no-check >> $S 2>&1
  DCI_GATHER_SERIAL=0 DCI_TMA_WARPS=2 DCI_TMA_SMEM_KB=100 bash tools/sweep.sh "tma_conc_w2_100" --inflight $inf --steps 300 --no-check >> $S 2>&1
done
cat $S
