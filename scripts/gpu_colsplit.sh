#!/bin/bash
export PATTN_LIB=$PWD/variants/colsplit/libpattn.so
timeout 60 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_tensor_core_path" 2>&1 | tail -3
timeout 60 python bench.py --streams 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('colsplit prefill', round(d['kernel_ms']['prefill']*1e3,1), 'us', round(d['roofline_kernels']['prefill']['achieved'],1), 'TF')"
