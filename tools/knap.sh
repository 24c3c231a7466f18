timeout 300 python -m pytest tests/test_gpu_random.py -m gpu -q -x -k knapsack 2>&1 | tail -1
for fan in 2,2,2 8,4,2 15,10,5; do for fill in dci knapsack; do for rep in 1 2; do timeout 300 python bench.py --config M3 --fanouts $fan --fill $fill --no-cpu-baseline --no-check --repeats 1 --steps 300 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stats']
print('$fan $fill', '%.3f M/s'%(d['value']/1e6), 'adj %.3f feat %.3f'%(s['adj_hit_rate'],s['feat_hit_rate']), 'C_adj %.1f MB C_feat %.1f MB'%(s['c_adj']/1e6,s['c_feat']/1e6), 'fill %.3f s presample %.3f s'%(s['preprocess_s']['fill'], s['preprocess_s']['presample']))"; done; done; done
