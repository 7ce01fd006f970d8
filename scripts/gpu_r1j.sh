#!/bin/bash
LIBS="main onemma" bash scripts/gpu_k1_ab.sh
PATTN_LIB=$PWD/variants/trace/libpattn.so timeout 100 python scripts/k1_trace.py > gpurun_out/k1_trace_sm.txt 2>&1; grep -E "softmax a dur|phases|MMA gap|Q ready|SMa_start " gpurun_out/k1_trace_sm.txt
