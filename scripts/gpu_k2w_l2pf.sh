#!/bin/bash
# K2W L2 prefetch of K/V boxes PATTN_K2W_L2PF sub-blocks ahead of the ring (variants pf4/8/16) vs main.
run() {  # lib workload streams [env]
  if [ $1 == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$1/libpattn.so; fi
  timeout 200 python bench.py --workload $2 --streams $3 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_ms']
print('$1 $2 ${PATTN_DECODE_SMS:-} step %.1f us' % (d['ms_per_step']*1e3), 'decode %.1f' % (k['decode']*1e3))"
}
for rep in 1 2; do
  for L in main pf4 pf8 pf16; do
    run $L c3_mixed8b 2
    run $L c2_decode8b 2
    PATTN_DECODE_SMS=36 run $L c3d_decode_part 1
  done
done
for L in main pf8; do run $L c4_decode128k 2; run $L c5_mixed70b 2; done
PATTN_LIB=$PWD/variants/pf8/libpattn.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "decode_wide or k2w_matrix or full_size or needle" 2>&1 | tail -1
