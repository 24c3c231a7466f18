timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/exp4_tests.txt
S=gpurun_out/exp4_sweep.txt
bash tools/sweep.sh "single" --inflight 6 --steps 300 --no-check >> $S 2>&1
for g in 2 3 6; do for inf in 2 3; do
  bash tools/sweep.sh "group$g" --group $g --inflight $inf --steps 300 --no-check >> $S 2>&1
done; done
DCI_GATHER_SERIAL=0 bash tools/sweep.sh "group3_conc" --group 3 --inflight 3 --steps 300 --no-check >> $S 2>&1
DCI_TMA_WARPS=8 bash tools/sweep.sh "group3_w8" --group 3 --inflight 2 --steps 300 --no-check >> $S 2>&1
DCI_TMA_SMEM_KB=100 DCI_TMA_WARPS=2 bash tools/sweep.sh "group3_w2_100" --group 3 --inflight 2 --steps 300 --no-check >> $S 2>&1
cat gpurun_out/exp4_tests.txt $S
