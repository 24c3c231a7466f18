# session 3: TIMING ONLY -- the sweeping hop without its atomicMax insertions (DCI_PRECHECK=9, wrong results), an upper bound on what filtering no-op atomics could save
mkdir -p gpurun_out/r3o; rm -rf gpurun_out/r3o/*
for c in 0 9; do DCI_PRECHECK=$c bash tools/exp/launches.sh na$c --steps 20 --warmup 5; done
cp gpurun_out/exp/launches_na*.csv gpurun_out/r3o/
