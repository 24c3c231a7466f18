timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/exp17_tests.txt
cat gpurun_out/exp17_tests.txt
S=gpurun_out/exp17_sweep.txt
run() { lab=$1; shift; env bash tools/sweep.sh "$lab" --steps 480 --no-check "$@" >> $S 2>&1; }
run g6i3 --group 6 --inflight 3
run g8i3 --group 8 --inflight 3
run g12i2 --group 12 --inflight 2
run g4i3 --group 4 --inflight 3
run single --group 0 --inflight 6
run M1_g6i3 --config M1 --group 6 --inflight 3
run M1_g16i3 --config M1 --group 16 --inflight 3
cat $S
