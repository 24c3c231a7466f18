S=gpurun_out/exp19_sweep.txt
run() { lab=$1; shift; a=(); e=(); for x in "$@"; do case $x in DCI_*) e+=("$x");; *) a+=("$x");; esac; done; env "${e[@]}" bash tools/sweep.sh "$lab" --steps 480 --no-check "${a[@]}" >> $S 2>&1; }
for c in M3 M4s; do
run ${c}_single --config $c --group 0 --inflight 6
run ${c}_g6i3 --config $c --group 6 --inflight 3
run ${c}_g4i4 --config $c --group 4 --inflight 4
run ${c}_g6i3_conc --config $c --group 6 --inflight 3 DCI_GATHER_SERIAL=0
done
cat $S
