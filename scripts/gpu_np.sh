#!/bin/bash
# K2 producer-warp count (PATTN_K2_NP) A/B
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for L in main np3 np4; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "long_decode or needle" 2>&1 | tail -1
  timeout 120 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "$L"
  for c in 1 2; do PATTN_DECODE_SMS=36 PATTN_DECODE_CTAS=$c timeout 120 python bench.py --workload c3d_decode_part --streams 1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "$L sm36 ctas$c"; done
  timeout 120 python bench.py --workload c2_decode8b --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "$L"
done
