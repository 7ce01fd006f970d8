#!/bin/bash
# K1 FMA-pipe exponential share (PATTN_K1_POLY pairs of 8) x tile size: parity subset + serial prefill time.
mkdir -p gpurun_out
for L in ${LIBS:-main poly2 poly4}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  for T in ${TILES:-64 128}; do
    PATTN_K1_TILE=$T timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill or random_mixed or needle" 2>&1 | tail -1
    for W in ${WS:-c3p_prefill_part}; do
      PATTN_K1_TILE=$T timeout 200 python bench.py --workload $W --streams 1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline_kernels']
print('$L tile $T $W step %.1f us' % (d['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()},
      {k: (round(v['achieved'],1), round(v['frac'],3)) for k,v in r.items()})"
    done
  done
done
echo "=== trace poly4 tile 128"
PATTN_K1_TILE=128 PATTN_LIB=$PWD/variants/trace_poly4/libpattn.so timeout 120 python scripts/k1_trace.py > gpurun_out/trace_p4_128.txt 2>&1; grep -v "^ *[0-9]* " gpurun_out/trace_p4_128.txt | tail -22
echo "=== trace poly4 tile 64"
PATTN_K1_TILE=64 PATTN_LIB=$PWD/variants/trace_poly4/libpattn.so timeout 120 python scripts/k1_trace.py > gpurun_out/trace_p4_64.txt 2>&1; grep -v "^ *[0-9]* " gpurun_out/trace_p4_64.txt | tail -22
