#!/bin/bash
for d in variants/tr_*/; do
  echo "== $d"; PATTN_LIB=$PWD/$d/libpattn.so timeout 120 python scripts/k1_trace.py 2>&1 | grep -E "softmax a duration|^SMa_start +n="
done
