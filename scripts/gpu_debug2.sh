#!/bin/bash
mkdir -p gpurun_out
export PATTN_DECODE_WARPS=4 PATTN_DECODE_CTAS=2 PATTN_DECODE_RING_KB=64
timeout 60 python scripts/one_call.py c2_decode8b 3 2>&1 | tail -3
timeout 300 compute-sanitizer --tool memcheck python scripts/one_call.py c2_decode8b 1 16x4096:1 2>&1 | grep -v "^=========     " | head -40
timeout 300 compute-sanitizer --tool synccheck python scripts/one_call.py c2_decode8b 1 16x4096:1 2>&1 | head -20
timeout 600 compute-sanitizer --tool racecheck --racecheck-report analysis python scripts/one_call.py c2_decode8b 1 4x4096:1 2>&1 | head -30
