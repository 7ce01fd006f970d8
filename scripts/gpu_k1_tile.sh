#!/bin/bash
# K1 tile-size A/B: 64-key (double-buffered S) vs 128-key ping-pong schedule.
#   parity subset under PATTN_K1_TILE=128, then serial prefill time on c3p / c3 for both tiles.
mkdir -p gpurun_out
PATTN_K1_TILE=128 timeout ${PT:-300} python -m pytest tests/test_gpu_parity.py -x -q -k "${TESTS:-prefill or random_mixed or needle}" 2>&1 | tail -${TAILN:-3}
for T in ${TILES:-64 128}; do
  for W in ${WS:-c3p_prefill_part c3_mixed8b}; do
    PATTN_K1_TILE=$T timeout 200 python bench.py --workload $W --streams ${STREAMS:-1} --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('tile $T $W step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"
  done
done
