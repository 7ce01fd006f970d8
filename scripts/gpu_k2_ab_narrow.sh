#!/bin/bash
# K2 (narrow) under the K2W-measured tuning leaf: its own defaults must apply (decode_kernel 2 via env).
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "decode or needle or split or random or tuning" 2>&1 | tail -1
for K in 0 1; do
  for W in c2_decode8b c4_decode128k c3_mixed8b; do
    PATTN_DECODE_WIDE=$K timeout 120 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('wide$K', d['config']['workload'], round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
  done
done
