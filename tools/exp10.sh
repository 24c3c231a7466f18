S=gpurun_out/exp10_sweep.txt
run() { lab=$1; g=$2; inf=$3; shift 3; env "$@" bash tools/sweep.sh "$lab" --group $g --inflight $inf --steps 384 --no-check >> $S 2>&1; }
run g8i3 8 3
run g8i3_sbps4 8 3 DCI_SAMPLE_BPS=4
run g8i3_sbps2 8 3 DCI_SAMPLE_BPS=2
run g8i3_sbps1 8 3 DCI_SAMPLE_BPS=1
run g8i3_prio 8 3 DCI_SAMPLE_PRIO=1
run g4i4_sbps2 4 4 DCI_SAMPLE_BPS=2
run g6i3_sbps2 6 3 DCI_SAMPLE_BPS=2
cat $S
