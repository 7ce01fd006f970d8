#!/bin/bash
# Build libpattn with extra defines into variants/<name>/libpattn.so (A/B and trace builds;
# select at run time with PATTN_LIB=variants/<name>/libpattn.so).
#   bash scripts/build_variant.sh trace -DPATTN_TRACE
set -e
name=$1; shift
cd "$(dirname "$0")/.."
SRC=${SRC:-paper_2511_11581_b200/csrc}
mkdir -p variants/$name/build
objs=""
for f in pattn_api k5_metadata k4_generic k2_decode k2w_decode k3_reduce k1_prefill k6_write_kv k7_baseline; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr -Iinclude -I$SRC \
    -DPATTN_BUILD "$@" -c $SRC/$f.cu -o variants/$name/build/$f.o &
  objs="$objs variants/$name/build/$f.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libpattn.so $objs \
  -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64
echo built variants/$name/libpattn.so
