#!/bin/bash
# mixed-batch knobs: decode consumer warps, K1 cost-model constant of the two-stream partition
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'P', d['roofline_kernels'].get('prefill',{}).get('prefill_sms'), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for W in c3_mixed8b; do
  for dw in 4 8; do
    for t in 2.2 2.5 2.8 3.1; do
      PATTN_DECODE_WARPS=$dw PATTN_K1_TILE_US=$t timeout 200 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "warps$dw tile$t"
    done
  done
done
for t in 2.2 2.5 2.8; do
  PATTN_K1_TILE_US=$t timeout 200 python bench.py --workload c5_mixed70b --shard seq --sim-world 8 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "tile$t"
done
