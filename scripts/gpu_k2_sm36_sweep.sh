#!/bin/bash
# K2 per-SM streaming rate on 36 SMs (the mixed step's decode share): consumer warps x CTAs/SM x ring.
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['kernel_ms']['decode']
print('$1', d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), 'decode', round(t*1e3,1), 'us', round(0.9407/t/36*1e3,1), 'GB/s/SM')"; }
for w in 4 8; do for c in 1 2 3; do for r in 64 96 192; do
  PATTN_DECODE_WARPS=$w PATTN_DECODE_CTAS=$c PATTN_DECODE_RING_KB=$r PATTN_DECODE_SMS=36 timeout 120 python bench.py --workload c3d_decode_part --streams 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "ncw$w ctas$c ring$r"
done; done; done
