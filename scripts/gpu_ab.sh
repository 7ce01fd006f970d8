#!/bin/bash
# A/B of library variants: parity subset + per-workload step and per-kernel times.
#   LIBS="main v1" WS="c3_mixed8b c2_decode8b" STREAMS=2 bash scripts/gpu_ab.sh
for L in ${LIBS:-main}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  [ -n "$NOTEST" ] || timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "${TESTS:-prefill or random_mixed or needle or long_decode}" 2>&1 | tail -1
  for W in ${WS:-c3_mixed8b}; do
    timeout 300 python bench.py --workload $W --streams ${STREAMS:-2} --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('$L $W step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"
  done
done
