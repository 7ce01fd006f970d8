#!/bin/bash
# Config 3: decode-side knobs in the mixed step (K2W ring size, heads per box, partition rate).
run() {
  timeout 200 python bench.py --workload c3_mixed8b --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_ms']
print('$1 step %.1f us' % (d['ms_per_step']*1e3), 'prefill %.1f decode %.1f' % (k['prefill']*1e3, k['decode']*1e3))"
}
for rep in 1 2; do
  run base
  PATTN_DECODE_RING_KB=192 run ring192
  PATTN_DECODE_RING_KB=160 run ring160
  PATTN_DECODE_WIDE_HB=4 run hb4
  PATTN_K2W_SM_GBS=110 run rate110
  PATTN_K2W_SM_GBS=90 run rate90
  PATTN_ITEMS_PER_SM=3 run ips3
done
