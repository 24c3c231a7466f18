#!/bin/bash
# bench sweep helper: prints one summary line per run.  Usage: tools/sweep.sh "<label>" <bench args...>
label=$1; shift
timeout 400 python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; s=d['stats']
print('$label', 'inflight', d['config']['inflight'], 'frac %.3f' % r['frac'], 'alone %s' % (('%.3f' % r['alone']['frac']) if r.get('alone') else '-'), '%.3f Mseeds/s' % (d['value']/1e6), 'gather %.0f GB/s %.4f ms agg %.0f GB/s' % (r['achieved'], r['avg_gather_ms'], r['aggregate_achieved']), 'sample %.4f ms' % r['avg_sample_ms'], 'e2e %.3f' % (d['e2e']['value']/1e6), 'host %.3f ms/step' % s['host_enqueue_ms_per_step'], 'adj_hit %.3f feat_hit %.3f' % (s['adj_hit_rate'], s['feat_hit_rate']))
"
