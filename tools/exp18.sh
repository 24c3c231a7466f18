S=gpurun_out/exp18_sweep.txt
run() { lab=$1; shift; env "$@" bash tools/sweep.sh "$lab" --steps 480 --no-check $ARGS >> $S 2>&1; }
for b in 3 4 8; do
ARGS="--group 6 --inflight 3" run g6i3_b$b DCI_SAMPLE_BPS=$b
ARGS="--group 8 --inflight 3" run g8i3_b$b DCI_SAMPLE_BPS=$b
ARGS="--group 6 --inflight 2" run g6i2_b$b DCI_SAMPLE_BPS=$b
done
cat $S
