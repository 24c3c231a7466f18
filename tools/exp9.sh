./tools/probe/hbm_gather_probe | grep -v '"seq"\|"sorted"' > gpurun_out/exp9_probe.txt
S=gpurun_out/exp9_sweep.txt
bash tools/sweep.sh "g8i1" --group 8 --inflight 1 --steps 384 --no-check >> $S 2>&1
bash tools/sweep.sh "g4i1" --group 4 --inflight 1 --steps 384 --no-check >> $S 2>&1
DCI_TMA_CHUNK=2400 bash tools/sweep.sh "g8i1_r1" --group 8 --inflight 1 --steps 384 --no-check >> $S 2>&1
DCI_TMA_CHUNK=2400 DCI_TMA_WARPS=16 bash tools/sweep.sh "g8i1_r1w16" --group 8 --inflight 1 --steps 384 --no-check >> $S 2>&1
cat gpurun_out/exp9_probe.txt $S
