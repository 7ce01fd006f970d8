#!/bin/bash
# Mixed steps (two streams) vs the partition model's decode-rate constant (PATTN_K2W_SM_GBS).
two() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for G in ${GBS:-80 100 120}; do for W in ${WS:-c3_mixed8b}; do
  PATTN_K2W_SM_GBS=$G timeout 120 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | two "gbs$G"
done; done
