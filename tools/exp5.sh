S=gpurun_out/exp5_sweep.txt
run() { lab=$1; shift; env "$@" bash tools/sweep.sh "$lab" --group 3 --inflight 2 --steps 300 --no-check >> $S 2>&1; }
run w8 DCI_TMA_WARPS=8
run w12 DCI_TMA_WARPS=12
run w16 DCI_TMA_WARPS=16
run w16_220 DCI_TMA_WARPS=16 DCI_TMA_SMEM_KB=220
run w8_4k DCI_TMA_WARPS=8 DCI_TMA_CHUNK=4096
run w16_4k DCI_TMA_WARPS=16 DCI_TMA_CHUNK=4096
run w16_2k DCI_TMA_WARPS=16 DCI_TMA_CHUNK=2048
run w8x2 DCI_TMA_WARPS=8 DCI_TMA_SMEM_KB=110 DCI_TMA_BPS=2
run w8_conc DCI_TMA_WARPS=8 DCI_GATHER_SERIAL=0
run w16_conc DCI_TMA_WARPS=16 DCI_GATHER_SERIAL=0
env DCI_TMA_WARPS=16 bash tools/sweep.sh "w16_g6" --group 6 --inflight 2 --steps 300 --no-check >> $S 2>&1
env DCI_TMA_WARPS=16 bash tools/sweep.sh "w16_g2" --group 2 --inflight 3 --steps 300 --no-check >> $S 2>&1
cat $S
