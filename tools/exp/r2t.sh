# does aligning X rows to 512 B / 1 KB help the random-row write pattern? (scatter probe)
mkdir -p gpurun_out/r2t
for P in 2432 2560 3072 2048 4096; do
timeout 300 ./tools/probe/scatter_probe 232965 $P 141187 20 > gpurun_out/r2t/scatter_$P.jsonl 2>&1
done
