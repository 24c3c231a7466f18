timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/exp8_tests.txt
cat gpurun_out/exp8_tests.txt
S=gpurun_out/exp8_sweep.txt
run() { lab=$1; g=$2; inf=$3; shift 3; env "$@" bash tools/sweep.sh "$lab" --group $g --inflight $inf --steps 384 --no-check >> $S 2>&1; }
bash tools/sweep.sh "single" --inflight 6 --steps 384 --no-check >> $S 2>&1
run g2i3 2 3
run g4i2 4 2
run g4i3 4 3
run g8i2 8 2
run g8i3 8 3
run g8i2_w16 8 2 DCI_TMA_WARPS=16
run g6i2 6 2
cat $S
