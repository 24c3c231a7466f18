timeout 900 python -m pytest tests/test_gpu_many.py -q -x 2>&1 | tail -3 > gpurun_out/exp16_tests.txt
S=gpurun_out/exp16_sweep.txt
run() { lab=$1; shift; env bash tools/sweep.sh "$lab" --steps 480 --no-check "$@" >> $S 2>&1; }
run g6i3 --group 6 --inflight 3
run g8i3 --group 8 --inflight 3
run g10i2 --group 10 --inflight 2
run g12i2 --group 12 --inflight 2
run g16i2 --group 16 --inflight 2
run g12i3 --group 12 --inflight 3
run g16i3 --group 16 --inflight 3
cat gpurun_out/exp16_tests.txt $S
