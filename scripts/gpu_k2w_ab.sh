#!/bin/bash
# K2W A/B: decode tests, per-SM rate on 36 SMs, configs 2/4 and the mixed config 3.
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['kernel_ms']['decode']
print('$1', 'decode', round(t*1e3,1), 'us', round(0.9407/t/36*1e3,1), 'GB/s/SM')"; }
two() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "decode or needle or split or gather or full_size" 2>&1 | tail -1
for L in ${LIBS:-main}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  PATTN_DECODE_SMS=36 timeout 120 python bench.py --workload c3d_decode_part --streams 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "$L sm36"
  for W in c2_decode8b c4_decode128k c3_mixed8b; do
    timeout 120 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | two "$L"
  done
done
