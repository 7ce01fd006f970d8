#!/bin/bash
# A/B of library variants on full bench lines (eager + CUDA-graph replay), no sub-results.
for L in ${LIBS:-main}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  for W in ${WS:-c3_mixed8b}; do
    timeout 300 python bench.py --workload $W --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']; g=d.get('cuda_graph') or {}
print('$L $W step %.1f us graph %.1f us' % (d['ms_per_step']*1e3, (g.get('ms_per_step') or 0)*1e3),
      {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, r.get('prefill',{}).get('prefill_sms'))"
  done
done
