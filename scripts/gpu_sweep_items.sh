#!/bin/bash
# decode segment-count sweep (PATTN_TARGET_ITEMS) on configs 2, 3, 4
for wl in c3_mixed8b c2_decode8b c4_decode128k; do
  for t in 1184 2368 3552 4736 7104; do
    r=$(PATTN_TARGET_ITEMS=$t timeout 120 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1),'us step', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})")
    echo "$wl target_items=$t: $r"
  done
done
