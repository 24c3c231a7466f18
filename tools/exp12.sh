S=gpurun_out/exp12_sweep.txt
run() { lab=$1; shift; bash tools/sweep.sh "$lab" --steps 384 --no-check "$@" >> $S 2>&1; }
run g6i3 --group 6 --inflight 3
run g6i3_line --group 6 --inflight 3 --ldx line
run g8i3_line --group 8 --inflight 3 --ldx line
run g4i4_line --group 4 --inflight 4 --ldx line
run single_line --group 0 --inflight 6 --ldx line
cat $S
