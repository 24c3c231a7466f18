# sweep gather knobs at K=20: L2 hint, ring shape
mkdir -p gpurun_out/r2ee
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-check --no-aggregate > gpurun_out/r2ee/$tag.json 2> gpurun_out/r2ee/$tag.log; }
run base
run hint0 DCI_TMA_HINT=0
run w4k8 DCI_SWEEP_WARPS=4 DCI_SWEEP_SLOTS=8
run w8k2 DCI_SWEEP_WARPS=8 DCI_SWEEP_SLOTS=2
run w8k6 DCI_SWEEP_WARPS=8 DCI_SWEEP_SLOTS=6
run base2
