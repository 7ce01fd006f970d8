#!/bin/bash
# K2 one-ahead scores (PIPE) needs spare stages: try it with large rings (ctas=1) on mixed batches.
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for cfg in "0 96" "1 192" "0 192" "1 144"; do set -- $cfg
  PATTN_K2_PIPE=$1 PATTN_DECODE_RING_KB=$2 timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "pipe$1 ring$2"
  PATTN_K2_PIPE=$1 PATTN_DECODE_RING_KB=$2 PATTN_DECODE_SMS=36 PATTN_DECODE_CTAS=1 timeout 120 python bench.py --workload c3d_decode_part --streams 1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "pipe$1 ring$2 sm36"
done
