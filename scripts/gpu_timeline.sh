#!/bin/bash
export PATTN_LIB=$PWD/variants/trace/libpattn.so
echo "== c2 decode on 16 SMs"; PATTN_DECODE_SMS=16 timeout 120 python scripts/timeline.py c2_decode8b 1 2>&1 | grep -v "^  " | tail -8
echo "== c2 decode full"; timeout 120 python scripts/timeline.py c2_decode8b 1 2>&1 | grep -v "^  " | tail -8
echo "== c3 2 streams P=108"; PATTN_PREFILL_SMS=108 timeout 120 python scripts/timeline.py c3_mixed8b 2 2>&1 | tail -40
echo "== c3 serial"; timeout 120 python scripts/timeline.py c3_mixed8b 1 2>&1 | tail -40
