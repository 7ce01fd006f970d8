#!/bin/bash
# Two-stream SM partition sweep: K1 grid = PATTN_PREFILL_SMS, decode fills the rest.
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
W=${1:-c3_mixed8b}
line() {
python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
g=d.get('cuda_graph') or {}
print('$1', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, 'graph', round(g.get('ms_per_step',0)*1e3,1), g.get('replay_matches_eager'))"
}
DCS=${DCS:-2,96}
for DC in $DCS; do
  set -- $(echo $DC | tr ',' ' ')
  for P in ${PS:-0 96 104 112 120 128}; do
    PATTN_DECODE_CTAS=$1 PATTN_DECODE_RING_KB=$2 PATTN_PREFILL_SMS=$P timeout 200 python bench.py --workload $W --streams 2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | line "ctas $1 ring $2 P $P"
  done
  PATTN_DECODE_CTAS=$1 PATTN_DECODE_RING_KB=$2 timeout 200 python bench.py --workload $W --streams 1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | line "serial ctas $1 ring $2"
done
for W2 in c2_decode8b c4_decode128k; do
  timeout 200 python bench.py --workload $W2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | line "$W2"
done
