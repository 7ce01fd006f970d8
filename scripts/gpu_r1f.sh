#!/bin/bash
mkdir -p gpurun_out
LIBS="main nopp" bash scripts/gpu_k1_ab.sh
PATTN_LIB=$PWD/variants/trace/libpattn.so timeout 100 python scripts/k1_trace.py > gpurun_out/k1_trace_pp.txt 2>&1; grep -E "softmax a|SMa_start|MMA gap|phases" gpurun_out/k1_trace_pp.txt
