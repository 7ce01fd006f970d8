#!/bin/bash
export PATTN_LIB=$PWD/variants/trace/libpattn.so
for DC in 3,64 2,96 1,192 4,48; do
  set -- $(echo $DC | tr ',' ' ')
  echo "== c2 decode on 16 SMs ctas $1 ring $2"; PATTN_DECODE_CTAS=$1 PATTN_DECODE_RING_KB=$2 PATTN_DECODE_SMS=16 timeout 120 python scripts/timeline.py c2_decode8b 1 2>&1 | grep -E "k2|items"
done
