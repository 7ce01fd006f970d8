#!/bin/bash
mkdir -p gpurun_out
export PATTN_DECODE_WIDE=1
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --error-exitcode 3 python scripts/one_call.py c3_mixed8b 1 "2x700:1+1x0:200" 2>&1 | tail -30 > gpurun_out/k2w_racecheck.txt; tail -12 gpurun_out/k2w_racecheck.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -k "not sanitizer" 2>&1 | tail -4
one() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('$1', d['config']['workload'], 'step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for W in c2_decode8b c4_decode128k; do for I in 4 8 16; do
  PATTN_WIDE_ITEMS_PER_SM=$I timeout 120 python bench.py --workload $W --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "items$I"
done; done
for G in 90 110 130 150; do
  PATTN_K2W_SM_GBS=$G timeout 120 python bench.py --workload c3_mixed8b --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | one "gbs$G"
done
