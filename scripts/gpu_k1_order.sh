#!/bin/bash
# K1 claim order A/B: rank-major (uniform Q-block batches) vs per-sequence; CTA end spread (trace).
LIBS="main prev main prev" WS="c3p_prefill_part c3_mixed8b c5_mixed70b" NOTEST=1 bash scripts/gpu_k1_ab.sh
PATTN_LIB=$PWD/variants/trace/libpattn.so timeout 120 python scripts/graph_timeline.py c3_mixed8b 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill or random_mixed or needle or gather or full_size or partition" 2>&1 | tail -2
