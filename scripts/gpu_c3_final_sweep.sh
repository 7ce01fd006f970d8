#!/bin/bash
# Config 3 / 5 around the session-4 defaults: claim-group budget x fixed SM split.
run() {
  timeout 200 python bench.py --workload $1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1 mb=${PATTN_K1_GROUP_MB:-def} P=${PATTN_PREFILL_SMS:-model} step %.1f us' % (d['ms_per_step']*1e3))"
}
for rep in 1 2; do
  run c3_mixed8b
  PATTN_K1_GROUP_MB=64 run c3_mixed8b
  PATTN_K1_GROUP_MB=16 run c3_mixed8b
  for P in 116 122; do PATTN_PREFILL_SMS=$P run c3_mixed8b; done
  run c5_mixed70b
  PATTN_K1_GROUP_MB=16 run c5_mixed70b
  PATTN_K1_GROUP_MB=8 run c5_mixed70b
done
