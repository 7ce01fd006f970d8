#!/bin/bash
# Two-stream partition model constant (K2 per-SM rate) x decode CTAs per SM, mixed batches.
for W in c3_mixed8b; do
for g in 40 50 61 75; do for c in 1 2; do
  PATTN_K2_SM_GBS=$g PATTN_DECODE_CTAS=$c timeout 120 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$W gbs $g ctas $c step', round(d['ms_per_step']*1e3,1), 'P', d['roofline_kernels']['prefill']['prefill_sms'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
done; done; done
for g in 40 61; do for c in 1 2; do
  PATTN_K2_SM_GBS=$g PATTN_DECODE_CTAS=$c timeout 120 python bench.py --workload c5_mixed70b --shard seq --sim-world 8 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5seq8 gbs $g ctas $c step', round(d['ms_per_step']*1e3,1), 'P', d['roofline_kernels']['prefill']['prefill_sms'])"
done; done
