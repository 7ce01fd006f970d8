#!/bin/bash
mkdir -p gpurun_out
PATTN_DECODE_WARPS=4 PATTN_DECODE_CTAS=2 PATTN_DECODE_RING_KB=64 timeout 100 python bench.py --workload c2_decode8b --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/dbg_a.json 2> gpurun_out/dbg_a.err; echo "rc=$?"; tail -5 gpurun_out/dbg_a.err
timeout 100 python bench.py --workload c4_decode128k --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/dbg_b.json 2> gpurun_out/dbg_b.err; echo "rc=$?"; tail -5 gpurun_out/dbg_b.err
timeout 240 python -m pytest tests/test_gpu_parity.py -x -v -k "not full_size" 2>&1 | grep -E "PASS|FAIL|ERROR|Timeout|rror" | head -60
