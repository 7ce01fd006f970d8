#!/bin/bash
LIBS="main nopp_f2fp" bash scripts/gpu_k1_ab.sh
PATTN_LIB=$PWD/variants/trace/libpattn.so timeout 100 python scripts/k1_trace.py > gpurun_out/k1_trace_q.txt 2>&1; grep -E "softmax a|items|Q ready|epilogue|period|PV wait" gpurun_out/k1_trace_q.txt
