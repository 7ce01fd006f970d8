#!/bin/bash
# K2W per-SM rate on 36 SMs and configs 2-4 / mixed 3.  (The no-load / no-compute ablations of
# DESIGN.md §6 K2W were variants built from patches with -DPATTN_K2W_NOLOAD / NOCOMPUTE, since removed.)
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['kernel_ms']['decode']
print('$1', 'decode', round(t*1e3,1), 'us', round(0.9407/t/36*1e3,1), 'GB/s/SM')"; }
run() { PATTN_DECODE_SMS=36 timeout 120 python bench.py --workload c3d_decode_part --streams 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "$1"; }
[ -n "$TESTS" ] && timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "$TESTS" 2>&1 | tail -2
run main
two() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for W in ${WS:-c2_decode8b c4_decode128k}; do timeout 120 python bench.py --workload $W --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | two main; done
for G in ${GBS:-80 100}; do
  PATTN_K2W_SM_GBS=$G timeout 120 python bench.py --workload c3_mixed8b --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | two "gbs$G"
done
