#!/bin/bash
LIBS="main k3v3full k4v3" bash scripts/gpu_k1_ab.sh
for t in 2.0 2.3 2.6 2.8; do
  for W in c3_mixed8b; do
  PATTN_K1_TILE_US=$t timeout 200 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tile_us $t $W step', round(d['ms_per_step']*1e3,1), 'P', d['roofline_kernels']['prefill']['prefill_sms'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
  done
  PATTN_K1_TILE_US=$t timeout 200 python bench.py --workload c5_mixed70b --shard seq --sim-world 8 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tile_us $t c5seq8 step', round(d['ms_per_step']*1e3,1), 'P', d['roofline_kernels']['prefill']['prefill_sms'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
done
