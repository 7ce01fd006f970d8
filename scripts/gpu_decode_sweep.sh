#!/bin/bash
# Decode kernel (K2) launch-shape sweep.  Every run is bounded.
mkdir -p gpurun_out
out=gpurun_out/decode_sweep.txt
: > $out
for wl in c2_decode8b c4_decode128k; do
  for cfg in "2 96" "2 64" "3 56" "3 72" "4 40" "1 160" "1 200"; do
    set -- $cfg
    r=$(PATTN_DECODE_CTAS=$1 PATTN_DECODE_RING_KB=$2 \
        timeout 120 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | \
        python -c "import json,sys
t=sys.stdin.read()
try:
  d=json.loads(t.strip().splitlines()[-1]); r=d['roofline_kernels']['decode']; print(round(r['kernel_ms']*1e3,1),'us',round(r['achieved']),'GB/s',round(r['frac'],3))
except Exception: print('FAIL', t[-300:].replace(chr(10),' | '))")
    echo "$wl ctas=$1 ring=$2KB: $r" | tee -a $out
  done
done
