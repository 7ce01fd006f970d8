#!/bin/bash
# K5 metadata A/B (closed-form tile count, 32-bit / float group arithmetic): launch-list K5 time
# and step times, library variants alternating.
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "partition or two_stream or claim_groups or large_batch or full_size or debug_plan" 2>&1 | tail -1
for L in main prev; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  for c in c3_mixed8b c2_decode8b; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k5_" -c 10 --csv --log-file gpurun_out/k5ab_${L}_$c.csv \
      python bench.py --workload $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > /dev/null 2>&1
    python -c "
import csv
r=[x for x in csv.reader(open('gpurun_out/k5ab_${L}_$c.csv')) if len(x)>10 and x[-3]=='gpu__time_duration.sum']
v=[float(x[-1]) for x in r]; print('$L $c k5 ncu', len(v), 'mean', round(sum(v)/len(v),3))"
  done
done
for L in main prev main prev; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  for W in c3_mixed8b c2_decode8b c5_mixed70b; do
    timeout 200 python bench.py --workload $W --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$L $W step %.1f us' % (d['ms_per_step']*1e3), 'metadata %.2f' % (d['kernel_ms']['metadata']*1e3))"
  done
done
