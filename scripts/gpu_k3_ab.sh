#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "long_decode or random_mixed or full_size or fused or needle" 2>&1 | tail -2
for L in main oldk3 main oldk3; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  for W in c2_decode8b c4_decode128k c3_mixed8b; do
    timeout 200 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', d['config']['workload'], 'step', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
  done
done
