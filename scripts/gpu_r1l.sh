#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "strided or canary" 2>&1 | tail -2
LIBS="main k3v3full main k3v3full" bash scripts/gpu_k1_ab.sh
PATTN_LIB=$PWD/variants/trace/libpattn.so timeout 100 python scripts/k1_trace.py > gpurun_out/k1_trace_b.txt 2>&1
