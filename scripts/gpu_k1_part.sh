#!/bin/bash
# Mixed step (c3) after the K1 claim-order change: fixed SM split P, items per SM, K1 tile cost.
run() {  # lib workload tag
  if [ $1 == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$1/libpattn.so; fi
  timeout 200 python bench.py --workload $2 --streams 2 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_ms']
print('$1 $2 $3 step', round(d['ms_per_step']*1e3,1), 'us', {a: round(b*1e3,1) for a,b in k.items()})"
}
for P in 112 116 118 120 122 124; do PATTN_PREFILL_SMS=$P run main c3_mixed8b P=$P; done
for P in 120 124 126; do PATTN_PREFILL_SMS=$P run prev c3_mixed8b P=$P; done
for i in 3 4 6; do for t in 2.4 2.8; do PATTN_ITEMS_PER_SM=$i PATTN_K1_TILE_US=$t run main c3_mixed8b ips=$i,tile=$t; done; done
for i in 3 4; do PATTN_ITEMS_PER_SM=$i run prev c3_mixed8b ips=$i; done
for i in 2 4; do for t in 2.4 2.8; do PATTN_ITEMS_PER_SM=$i PATTN_K1_TILE_US=$t run main c5_mixed70b ips=$i,tile=$t; done; done
run prev c5_mixed70b base
