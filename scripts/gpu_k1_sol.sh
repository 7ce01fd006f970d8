#!/bin/bash
# K1 speed-of-light experiments: prefill-kernel time with the softmax or the MMAs removed.
for L in ${LIBS:-main nomma nosm}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  timeout 200 python bench.py --workload ${W:-c3_mixed8b} --streams 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$L prefill', round(d['kernel_ms'].get('prefill',0)*1e3,1), 'us', 'clk', d['clocks'])"
done
