#!/bin/bash
# Mixed step (config 3, two streams): decode consumer warps x CTAs/SM x partition rate constant.
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'step', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for w in 4 8; do for c in 1 2 3; do for g in ${GBS:-61 90 120}; do
  PATTN_DECODE_WARPS=$w PATTN_DECODE_CTAS=$c PATTN_K2_SM_GBS=$g timeout 120 python bench.py --workload ${W:-c3_mixed8b} --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "ncw$w ctas$c gbs$g"
done; done; done
