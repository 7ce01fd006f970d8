#!/bin/bash
# K2 ring size per CTA (PATTN_DECODE_RING_KB) with the tree's CTA count, mixed and decode batches.
for kb in 96 144 200; do
  for W in c3_mixed8b c2_decode8b c4_decode128k; do
    PATTN_DECODE_RING_KB=$kb timeout 120 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ring $kb', d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
  done
  PATTN_DECODE_RING_KB=$kb timeout 120 python bench.py --workload c5_mixed70b --shard seq --sim-world 8 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ring $kb c5seq8 step', round(d['ms_per_step']*1e3,1))"
done
