#!/bin/bash
mkdir -p gpurun_out
for V in main noload; do
  if [ $V == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/k2w_$V/libpattn.so; fi
  PATTN_DECODE_SMS=36 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k2w_decode" -s 3 -c 1 -o gpurun_out/k2w_sm36_$V -f \
    python bench.py --workload c3d_decode_part --streams 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sub > gpurun_out/ncu_k2w_$V.log 2>&1
  ls -la gpurun_out/k2w_sm36_$V.ncu-rep
done
