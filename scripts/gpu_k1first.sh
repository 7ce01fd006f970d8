#!/bin/bash
# K1 launch-completion ordering of the decode stream: eager and CUDA-graph steps with / without.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "graph or two_stream or full_size or partition" 2>&1 | tail -1
two() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), 'graph %.1f us' % (d['cuda_graph']['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"; }
for rep in 1 2; do
for W in c3_mixed8b c5_mixed70b x_g7_mixed; do
  timeout 200 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | two "k1first"
  PATTN_NO_K1_FIRST=1 timeout 200 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | two "old"
done; done
