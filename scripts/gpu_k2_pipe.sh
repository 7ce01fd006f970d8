#!/bin/bash
# K2 A/B: scores of the next sub-block computed ahead (PATTN_K2_PIPE=1, default) vs not.
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for pipe in 1 0 1 0; do
  for W in c2_decode8b c4_decode128k c3_mixed8b; do
    PATTN_K2_PIPE=$pipe timeout 200 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "pipe$pipe"
  done
  PATTN_K2_PIPE=$pipe PATTN_DECODE_SMS=36 PATTN_DECODE_CTAS=1 timeout 200 python bench.py --workload c3d_decode_part --streams 1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "pipe$pipe sm36 ctas1"
done
