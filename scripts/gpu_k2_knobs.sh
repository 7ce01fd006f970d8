#!/bin/bash
# K2 consumer-warp count and ring size with 4 producers
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for cfg in "4 96" "8 96" "4 64" "4 112"; do set -- $cfg
  for W in c2_decode8b c4_decode128k c3_mixed8b; do
    PATTN_DECODE_WARPS=$1 PATTN_DECODE_RING_KB=$2 timeout 120 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "ncw$1 ring$2"
  done
  PATTN_DECODE_WARPS=$1 PATTN_DECODE_RING_KB=$2 PATTN_DECODE_SMS=36 PATTN_DECODE_CTAS=2 timeout 120 python bench.py --workload c3d_decode_part --streams 1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "ncw$1 ring$2 sm36"
done
