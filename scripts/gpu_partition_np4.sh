#!/bin/bash
for g in 58 61 66 72; do
  for W in c3_mixed8b; do
  PATTN_K2_SM_GBS=$g timeout 120 python bench.py --workload $W --steps 60 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$W gbs $g step', round(d['ms_per_step']*1e3,1), 'P', d['roofline_kernels']['prefill']['prefill_sms'])"
  done
  PATTN_K2_SM_GBS=$g timeout 120 python bench.py --workload c5_mixed70b --shard seq --sim-world 8 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5seq8 gbs $g step', round(d['ms_per_step']*1e3,1), 'P', d['roofline_kernels']['prefill']['prefill_sms'])"
done
