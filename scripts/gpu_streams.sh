#!/bin/bash
for st in 1 2; do
  timeout 200 python bench.py --streams $st --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('streams $st', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, 'graph', d.get('cuda_graph'))"
done
