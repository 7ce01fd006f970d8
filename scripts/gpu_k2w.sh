#!/bin/bash
# K2W (head-wide TMA boxes) vs K2: parity under PATTN_DECODE_WIDE=1, per-SM rate on 36 SMs, configs 2/3/4.
mkdir -p gpurun_out
PATTN_DECODE_WIDE=1 timeout ${PT:-600} python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -x -q 2>&1 | tail -${TAILN:-3}
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for WIDE in 0 1; do
  PATTN_DECODE_WIDE=$WIDE PATTN_DECODE_SMS=36 PATTN_DECODE_CTAS=1 timeout 120 python bench.py --workload c3d_decode_part --streams 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "wide$WIDE sm36"
  for W in ${WS:-c3_mixed8b c2_decode8b c4_decode128k}; do
    PATTN_DECODE_WIDE=$WIDE timeout 120 python bench.py --workload $W --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "wide$WIDE"
  done
done
