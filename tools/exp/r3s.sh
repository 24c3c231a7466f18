# session 3: single-rank runs over the node-shared adopted host graph (--shm-graph on): M1 with the
# oracle leg (features from the shared graph), M4 host memory with the graph pinned once
mkdir -p gpurun_out/r3s; rm -rf gpurun_out/r3s/*
timeout 600 python bench.py --config M1 --steps 20 --warmup 5 --shm-graph on > gpurun_out/r3s/m1_shm.json 2> gpurun_out/r3s/m1_shm.log
timeout 2000 python bench.py --config M4 --steps 40 --warmup 8 --check-light --no-cpu-baseline --shm-graph on > gpurun_out/r3s/m4_shm.json 2> gpurun_out/r3s/m4_shm.log
for f in gpurun_out/r3s/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', d['value'], d['e2e']['value'], d['config']['host_graph'], d.get('parity_check',{}).get('bit_exact'), d['stats']['preprocess_s']['generate'], d['stats']['preprocess_s']['load'], d['host_memory'])"; done
tail -3 gpurun_out/r3s/m4_shm.log
