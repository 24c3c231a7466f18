set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/exp1_tests.txt
for cfg in "def:" "ser1:DCI_GATHER_SERIAL=1 DCI_GATHER_BPS=1" "ser2:DCI_GATHER_SERIAL=1 DCI_GATHER_BPS=2" "ser3:DCI_GATHER_SERIAL=1 DCI_GATHER_BPS=3" "ser4:DCI_GATHER_SERIAL=1 DCI_GATHER_BPS=4"; do
  lab=${cfg%%:*}; envs=${cfg#*:}
  for inf in 6 10; do
    env $envs bash tools/sweep.sh "$lab" --inflight $inf --steps 300 --no-check >> gpurun_out/exp1_sweep.txt 2>&1
  done
done
cat gpurun_out/exp1_tests.txt gpurun_out/exp1_sweep.txt
