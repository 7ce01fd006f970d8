#!/bin/bash
# K1 A/B of library variants: prefill parity subset + serial prefill (c3p) and the mixed step (c3).
for L in ${LIBS:-main}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  [ -n "$NOTEST" ] || timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill or random_mixed or needle or gather" 2>&1 | tail -1
  for W in ${WS:-c3p_prefill_part c3_mixed8b}; do
    ST=2; [ $W == c3p_prefill_part ] && ST=1
    timeout 200 python bench.py --workload $W --streams $ST --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline_kernels'].get('prefill',{})
print('$L $W step', round(d['ms_per_step']*1e3,1), 'us prefill', round(d['kernel_ms'].get('prefill',0)*1e3,1), 'us', round(r.get('achieved',0),1), 'TFLOP/s')"
  done
done
