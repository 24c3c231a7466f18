mkdir -p gpurun_out/r2gg
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2gg/$tag.json 2> gpurun_out/r2gg/$tag.log; }
run base
run after DCI_EPI_AFTER=1
run b148 DCI_EPI_BLOCKS=148
run b74 DCI_EPI_BLOCKS=74
run base2
run after2 DCI_EPI_AFTER=1
