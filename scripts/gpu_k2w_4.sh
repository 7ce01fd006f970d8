#!/bin/bash
mkdir -p gpurun_out
export PATTN_DECODE_WIDE=1
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -3
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for I in 4 8 16; do for G in 90 110; do
  PATTN_WIDE_ITEMS_PER_SM=$I PATTN_K2W_SM_GBS=$G timeout 120 python bench.py --workload c3_mixed8b --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "items$I gbs$G"
done; done
for I in 4 8 16; do
  PATTN_WIDE_ITEMS_PER_SM=$I timeout 120 python bench.py --workload c5_mixed70b --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "items$I"
done
