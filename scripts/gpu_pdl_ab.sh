#!/bin/bash
# PDL A/B: the same library with PATTN_NO_PDL=1 (plain launches) and without (programmatic
# dependent launch), step time (plain region) and CUDA-graph replay.
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); g=d.get('cuda_graph') or {}
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), 'graph %.1f us' % ((g.get('ms_per_step') or 0)*1e3))"; }
for rep in 1 2; do for W in c2_decode8b c3_mixed8b c4_decode128k c1_tiny; do
  PATTN_NO_PDL=1 timeout 200 python bench.py --workload $W --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one nopdl
  timeout 200 python bench.py --workload $W --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one pdl
done; done
