#!/bin/bash
# Group-gather variants on M2 (round 2): env knobs; prints the gather launch time live and alone,
# and seeds/s.  Usage: gather_variants.sh "tag|ENV=.. ENV=..|bench args" ...
# Output: gpurun_out/exp/gather_variants.jsonl (appended)
mkdir -p gpurun_out/exp
out=gpurun_out/exp/gather_variants.jsonl
for spec in "$@"; do
  IFS='|' read -r tag envs bargs <<< "$spec"
  env $envs python bench.py --steps ${STEPS:-100} --warmup 20 --repeats 2 --no-cpu-baseline --no-check $bargs 2>/dev/null \
    | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']
print(json.dumps({'tag':'$tag','value':d['value'],'e2e':d['e2e']['value'],'gather_ms':r['avg_gather_ms'],'sample_ms':r['avg_sample_ms'],'alone_ms':(r['alone'] or {}).get('avg_gather_ms'),'frac':r['frac'],'busy':r['gather_busy_frac'],'ldx':d['config']['ldx'],'group':d['config']['group']}))" | tee -a $out
done
