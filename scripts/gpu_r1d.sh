#!/bin/bash
mkdir -p gpurun_out/tune
timeout 900 python scripts/tune.py --out gpurun_out/tune 2>&1 | tail -40
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_c3_def.json 2>gpurun_out/b_c3_def.err; tail -2 gpurun_out/b_c3_def.err
python -c "
import json; d=json.loads(open('gpurun_out/b_c3_def.json').read().strip().splitlines()[-1]); print(json.dumps(d['roofline'])); print(json.dumps(d['roofline_kernels']))"
