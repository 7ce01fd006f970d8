#!/bin/bash
two() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for I in ${ITEMS:-2 4}; do for G in ${GBS:-90 100 110}; do for W in ${WS:-c3_mixed8b}; do
  PATTN_WIDE_ITEMS_PER_SM=$I PATTN_K2W_SM_GBS=$G timeout 120 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | two "items$I gbs$G"
done; done; done
