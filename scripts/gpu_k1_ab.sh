#!/bin/bash
# K1 A/B: prefill-kernel time on c3 (serial) for library variants.
for L in ${LIBS:-main}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill or random_mixed or needle" 2>&1 | tail -1
  for W in ${WS:-c3_mixed8b}; do
    timeout 200 python bench.py --workload $W --streams 1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['roofline_kernels'].get('prefill',{})
print('$L $W step', round(d['ms_per_step']*1e3,1), 'us prefill', round(d['kernel_ms'].get('prefill',0)*1e3,1), 'us', round(k.get('achieved',0),1), 'TFLOP/s')"
  done
done
