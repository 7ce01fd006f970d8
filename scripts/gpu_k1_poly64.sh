#!/bin/bash
# K1 at D = 64: share of exponentials on the FMA pipe (PATTN_K1_POLY64 pairs of 8), serial prefill + mixed.
python - <<'PY' > /dev/null
PY
for L in main poly64_2 poly64_3 poly64_4 main; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "head_dim_64 or fuzz" 2>&1 | tail -1
  for W in x_d64_mixed; do
    for ST in 1 2; do
    timeout 120 python bench.py --workload $W --streams $ST --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline_kernels']
print('$L streams$ST', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()}, {k:(round(v['achieved']),round(v['frac'],3)) for k,v in r.items()})"
    done
  done
done
