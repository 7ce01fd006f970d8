#!/bin/bash
# Full verification of the committed tree on one B200: parity tests, then the quick bench/ncu pass.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
bash scripts/gpu_bench_quick.sh
