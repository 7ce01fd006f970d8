#!/bin/bash
mkdir -p gpurun_out
LIBS="main poly7 poly3 poly1" bash scripts/gpu_k1_ab.sh
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_c3_def.json 2>gpurun_out/b_c3_def.err; tail -2 gpurun_out/b_c3_def.err
python -c "
import json; d=json.loads(open('gpurun_out/b_c3_def.json').read().strip().splitlines()[-1]); print(json.dumps(d['roofline'])); print(json.dumps(d['roofline_kernels']))"
