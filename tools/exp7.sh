timeout 900 python -m pytest tests/test_gpu_many.py -x -q 2>&1 | tail -15 > gpurun_out/exp7_tests.txt
cat gpurun_out/exp7_tests.txt
S=gpurun_out/exp7_sweep.txt
run() { lab=$1; g=$2; inf=$3; shift 3; env "$@" bash tools/sweep.sh "$lab" --group $g --inflight $inf --steps 384 --no-check >> $S 2>&1; }
run g2i3 2 3
run g3i2 3 2
run g4i2 4 2
run g4i3 4 3
run g8i2 8 2
run g8i2_w4 8 2 DCI_TMA_WARPS=4
run g8i2_w16 8 2 DCI_TMA_WARPS=16
run g8i3 8 3
run g4i2_nosweep 4 2 DCI_SWEEP=0
cat $S
