#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
LIBS="main nopp_f2fp" bash scripts/gpu_k1_ab.sh
PATTN_K1_NO_TMA_STORE=1 timeout 200 python bench.py --workload c3_mixed8b --streams 1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('main no-tma-store prefill', round(d['kernel_ms']['prefill']*1e3,1))"
PATTN_LIB=$PWD/variants/trace/libpattn.so timeout 100 python scripts/k1_trace.py > gpurun_out/k1_trace_ts.txt 2>&1; grep -E "Q ready|epilogue|softmax a dur" gpurun_out/k1_trace_ts.txt
