S=gpurun_out/exp13_sweep.txt
run() { lab=$1; shift; bash tools/sweep.sh "$lab" --steps 384 --no-check "$@" >> $S 2>&1; }
for c in M1 M3 M4s; do
  run ${c}_single --config $c --group 0 --inflight 6
  run ${c}_g6i3 --config $c --group 6 --inflight 3
  run ${c}_g8i3 --config $c --group 8 --inflight 3
done
cat $S
