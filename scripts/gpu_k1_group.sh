#!/bin/bash
# K1 claim-group size (PATTN_K1_GROUP_MB) and partition model K1 cost (PATTN_K1_TILE_US) sweep.
run() {  # lib workload streams
  if [ $1 == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$1/libpattn.so; fi
  timeout 200 python bench.py --workload $2 --streams $3 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline_kernels'].get('prefill',{})
print('$1 $2 mb=${PATTN_K1_GROUP_MB:-64} tile=${PATTN_K1_TILE_US:-2.8} step', round(d['ms_per_step']*1e3,1), 'us prefill', round(d['kernel_ms'].get('prefill',0)*1e3,1), 'us', round(r.get('achieved',0),1), 'TFLOP/s')"
}
for mb in 8 16 32 64; do PATTN_K1_GROUP_MB=$mb run main c3p_prefill_part 1; done
run prev c5_mixed70b 2
for mb in 8 16 32 64; do PATTN_K1_GROUP_MB=$mb run main c5_mixed70b 2; done
for t in 2.8 2.6 2.4 2.2; do PATTN_K1_TILE_US=$t run main c3_mixed8b 2; done
run prev c3_mixed8b 2
for t in 2.6 2.4; do PATTN_K1_GROUP_MB=16 PATTN_K1_TILE_US=$t run main c5_mixed70b 2; done
for t in 2.6 2.4; do PATTN_K1_TILE_US=$t run prev c3_mixed8b 2; done
