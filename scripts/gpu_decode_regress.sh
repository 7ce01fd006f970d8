#!/bin/bash
# Why is K2 slower inside config 3 (serial) than on config 2?  A/B over library builds and workloads.
mkdir -p gpurun_out
one() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', d['config']['workload'], 'ms %.4f' % d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, 'sm', d['clocks']['sm_mhz'])
"; }
for L in main old6b7; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  for W in c3_mixed8b c3d_decode_part c2_decode8b; do
    timeout 200 python bench.py --workload $W --streams 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "$L s1"
  done
  timeout 200 python bench.py --workload c3_mixed8b --streams 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "$L s2"
done
unset PATTN_LIB
for c in 1 3; do PATTN_DECODE_CTAS=$c timeout 200 python bench.py --workload c3_mixed8b --streams 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | one "ctas$c s1"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"k2_" -c 6 --csv --log-file gpurun_out/ncu_k2_c3s1.csv python bench.py --workload c3_mixed8b --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_k2_c3s1.csv
