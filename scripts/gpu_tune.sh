#!/bin/bash
# Tuning sweep -> tree (results under gpurun_out/tune; copy the tree into the package afterwards).
mkdir -p gpurun_out/tune
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "decode or needle or split" 2>&1 | tail -2
timeout 3000 python scripts/tune.py --out gpurun_out/tune > gpurun_out/tune/tune.log 2>&1
tail -40 gpurun_out/tune/tune.log
