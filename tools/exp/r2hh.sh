mkdir -p gpurun_out/r2hh
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2hh/$tag.json 2> gpurun_out/r2hh/$tag.log; }
run base300
run after300 DCI_EPI_AFTER=1
run base300b
run after300b DCI_EPI_AFTER=1
run2() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2hh/$tag.json 2> gpurun_out/r2hh/$tag.log; }
run2 base20
run2 after20 DCI_EPI_AFTER=1
run2 base20b
run2 after20b DCI_EPI_AFTER=1
