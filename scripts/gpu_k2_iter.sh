#!/bin/bash
# K2 iteration: decode parity tests, per-CTA trace, c2/c4 bench, c3 partition sweep.
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
bash scripts/gpu_timeline2.sh
PS="${PS:-96 104 112 120}" bash scripts/gpu_partition.sh 2>&1 | grep -v passed
