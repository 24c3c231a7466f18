# sampling-hop occupancy: __launch_bounds__(256, mb) builds (build_exp/libdci_mb*.so) vs default
mkdir -p gpurun_out/r2m
for v in base mb5 mb6; do
  if [ $v = base ]; then L=paper_2503_01281_b200/libdci.so; else L=build_exp/libdci_$v.so; fi
  DCI_LIB=$PWD/$L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-check > gpurun_out/r2m/bench_$v.json 2> gpurun_out/r2m/bench_$v.log
  DCI_LIB=$PWD/$L bash tools/exp/launches.sh r2m_$v --steps 20 --warmup 5
done
