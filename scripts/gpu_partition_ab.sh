#!/bin/bash
for L in ${LIBS:-main np4}; do
  if [ $L == main ]; then unset PATTN_LIB; else export PATTN_LIB=$PWD/variants/$L/libpattn.so; fi
  echo "== $L"
  PS="${PS:-100 108 116 124 132}" bash scripts/gpu_partition.sh 2>&1 | grep -v passed
done
