#!/bin/bash
# A/B the K1 builds under variants/*/libpattn.so on config 3
for d in variants/*/; do
  r=$(PATTN_LIB=$PWD/$d/libpattn.so timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1),'us step', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, round(d['roofline_kernels']['prefill']['achieved'],1))")
  echo "$d: $r"
done
