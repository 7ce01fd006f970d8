#!/bin/bash
# Standalone decode A/B over library variants and launch shapes.
for L in ${LIBS:-main np1}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  for DC in ${DCS:-3,64 2,96 2,64 4,48}; do
    set -- $(echo $DC | tr ',' ' ')
    for W in c2_decode8b c4_decode128k; do
      PATTN_DECODE_CTAS=$1 PATTN_DECODE_RING_KB=$2 timeout 200 python bench.py --workload $W --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$L ctas $1 ring $2 $W decode', round(d['kernel_ms']['decode']*1e3,1), 'us', 'frac', round(d['roofline']['frac'],3))"
    done
  done
done
