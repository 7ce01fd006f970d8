#!/bin/bash
# Config 3: decode ring depth (1 decode CTA per SM, the tree's choice for mixed batches) x the
# partition model's per-SM decode rate (which moves SMs between K1 and K2).
for ring in 96 144 192; do for gbs in 61 75 90; do
  PATTN_DECODE_RING_KB=$ring PATTN_K2_SM_GBS=$gbs timeout 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline_kernels']
print('ring $ring k2gbs $gbs step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, 'P', r['prefill'].get('prefill_sms'))"
done; done
