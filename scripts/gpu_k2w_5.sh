#!/bin/bash
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for G in 60 75 90; do
  PATTN_K2W_SM_GBS=$G timeout 120 python bench.py --workload c5_mixed70b --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "gbs$G"
done
for G in 80 90 100; do
  PATTN_K2W_SM_GBS=$G timeout 120 python bench.py --workload c3_mixed8b --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "gbs$G"
done
for W in x_g7_mixed x_d64_mixed x_bs7_decode32k c1_tiny; do
  timeout 120 python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "wide-default"
  PATTN_DECODE_WIDE=0 timeout 120 python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "k2"
done
