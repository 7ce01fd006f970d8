#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "sanitizer" -rs 2>&1 | tail -3
export PATTN_DECODE_WIDE=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -k "not sanitizer" 2>&1 | tail -3
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for I in 2 4; do for G in 90 110 130; do
  PATTN_WIDE_ITEMS_PER_SM=$I PATTN_K2W_SM_GBS=$G timeout 120 python bench.py --workload c3_mixed8b --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "items$I gbs$G"
done; done
for W in c5_mixed70b c2_decode8b c4_decode128k; do for WIDE in 0 1; do
  PATTN_DECODE_WIDE=$WIDE timeout 120 python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "wide$WIDE"
done; done
