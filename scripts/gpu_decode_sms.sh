#!/bin/bash
# Per-SM decode throughput: c2 decode with the K2 grid limited to N SMs.
DCS=${DCS:-3,64 2,96 1,192 4,48}
for DC in $DCS; do
  set -- $(echo $DC | tr ',' ' ')
  for N in 16 48; do
    PATTN_DECODE_CTAS=$1 PATTN_DECODE_RING_KB=$2 PATTN_DECODE_SMS=$N timeout 200 python bench.py --workload c2_decode8b --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
t=d['kernel_ms']['decode']*1e-3; b=d['algorithmic']['kv_bytes'] if 'kv_bytes' in d.get('algorithmic',{}) else None
print('ctas $1 ring $2 sms $N decode_us', round(t*1e6,1), 'GB/s/SM', round(1.07e9/t/1e9/$N,1))"
  done
done
