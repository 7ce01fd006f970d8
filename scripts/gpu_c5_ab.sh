export PATTN_NO_TUNING_TREE=1 PATTN_ITEMS_PER_SM=4 PATTN_MIN_CHUNK_TOKENS=128 PATTN_DECODE_CTAS=1
NOTEST=1 LIBS="${LIBS:-r1 main r1 main}" WS="${WS:-c5_mixed70b c3_mixed8b}" bash scripts/gpu_ab_graph.sh
