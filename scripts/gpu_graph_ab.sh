#!/bin/bash
# Mixed steps eager vs CUDA-graph replay, library variants alternating.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "graph or two_stream or partition or full_size" 2>&1 | tail -1
for L in ${LIBS:-main prev main prev}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  for W in ${WS:-c3_mixed8b c5_mixed70b}; do
    timeout 200 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$L', d['config']['workload'], 'eager %.1f us' % (d['ms_per_step']*1e3), 'graph %.1f us' % (d['cuda_graph']['ms_per_step']*1e3), d['cuda_graph']['replay_matches_eager'])"
  done
done
