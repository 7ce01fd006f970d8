#!/bin/bash
PATTN_DECODE_CTAS=2 PATTN_DECODE_RING_KB=64 timeout 60 python scripts/one_call.py c2_decode8b 3 2>&1 | grep -E "^ok|WATCHDOG" | sort | awk '{print $0}' | head -400 > gpurun_out/wd.txt
wc -l gpurun_out/wd.txt
