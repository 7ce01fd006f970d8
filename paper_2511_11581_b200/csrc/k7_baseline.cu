// K7 -- the paper's BASELINE attention kernel, for didactic comparison (App. A,
// "Triton Baseline Attention Kernel").  Not on the default
// path: selected with PATTN_FLAG_BASELINE.
//
// As App. A describes it: one program instance per (query token, query head);
// the instance finds its KV head, its sequence by a binary search over the
// accumulated query lengths and its prefix length, loads its Q row and
// runs the tiled softmax of §4.1 over tiles of exactly BLOCK_SIZE keys, i.e.
// one paged KV block per tile.  Here an instance is one warp: lanes split the
// head dimension (D/32 elements each), a score is a warp-shuffle dot product, and the
// running (m, l, acc) stay in registers; the division is delayed to the end.
// No GQA packing, no Q blocks, no split-KV, no tensor cores: each K/V row is re-read by
// every query head and every query token that sees it -- the cost the paper's later
// optimisations remove.
#include "common.cuh"
#include "kernels.h"

namespace pattn {
namespace {

template <typename T>
__device__ __forceinline__ float ld_f32(const T* p);
template <>
__device__ __forceinline__ float ld_f32<float>(const float* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ float ld_f32<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(__ldg(p));
}
template <typename T>
__device__ __forceinline__ void st_from_f32(T* p, float x);
template <>
__device__ __forceinline__ void st_from_f32<float>(float* p, float x) {
  *p = x;
}
template <>
__device__ __forceinline__ void st_from_f32<__nv_bfloat16>(__nv_bfloat16* p, float x) {
  *p = __float2bfloat16_rn(x);
}
template <>
__device__ __forceinline__ float ld_f32<__half>(const __half* p) {
  return __half2float(__ldg(p));
}
template <>
__device__ __forceinline__ void st_from_f32<__half>(__half* p, float x) {
  *p = __float2half_rn(x);
}

template <typename T, int D>
__global__ void __launch_bounds__(128) k7_baseline(Params p) {
  constexpr int DV = D / 32;  // head-dim elements per lane: lane owns d = lane + 32 v
  const int lane = threadIdx.x & 31;
  const int64_t inst = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);  // (token, q head)
  if (inst >= (int64_t)p.T * p.Hq) return;
  const int tok = (int)(inst / p.Hq), h = (int)(inst % p.Hq);
  const int kvh = h / p.G;                                   // P:27 (contiguous GQA groups)
  const int b = upper_bound_minus1(p.cu_seqlens_q, p.B, tok);  // P:27-28 binary search
  const int q0 = p.cu_seqlens_q[b];
  const int qlen = p.cu_seqlens_q[b + 1] - q0;
  const int ctx = p.seq_lens[b] - qlen;
  const int n = ctx + (tok - q0) + 1;  // keys 0 .. ctx + i (self-inclusive prefix)
  const T* Q = static_cast<const T*>(p.q) + (int64_t)tok * p.q_st_tok + (int64_t)h * p.q_st_head;
  const T* K = static_cast<const T*>(p.k);
  const T* V = static_cast<const T*>(p.v);
  float q[DV], acc[DV];
#pragma unroll
  for (int v = 0; v < DV; ++v) {
    q[v] = ld_f32(Q + lane + 32 * v) * p.scale_log2;  // scores in the log2 domain
    acc[v] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const int32_t* bt = p.block_table + (int64_t)b * p.bt_stride;
  for (int t0 = 0; t0 < n; t0 += p.bs) {  // one tile = one KV block (tile size = BLOCK_SIZE)
    const int64_t blk = bt[t0 / p.bs];
    const int nt = min(p.bs, n - t0);
    // tile max first (the tiled softmax of P:249-257 updates once per tile)
    float mt = -INFINITY;
    for (int j = 0; j < nt; ++j) {
      const T* kr = K + blk * p.kv_st_blk + (int64_t)j * p.kv_st_tok + (int64_t)kvh * p.kv_st_head;
      float s = 0.f;
#pragma unroll
      for (int v = 0; v < DV; ++v) s = fmaf(q[v], ld_f32(kr + lane + 32 * v), s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      mt = fmaxf(mt, s);
    }
    const float mn = fmaxf(m, mt);
    const float alpha = exp2f(m - mn);  // m = -inf on the first tile: alpha = 0
    l *= alpha;
#pragma unroll
    for (int v = 0; v < DV; ++v) acc[v] *= alpha;
    for (int j = 0; j < nt; ++j) {  // scores recomputed: the baseline keeps no tile in memory
      const int64_t row = blk * p.kv_st_blk + (int64_t)j * p.kv_st_tok + (int64_t)kvh * p.kv_st_head;
      float s = 0.f;
#pragma unroll
      for (int v = 0; v < DV; ++v) s = fmaf(q[v], ld_f32(K + row + lane + 32 * v), s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const float pr = exp2f(s - mn);
      l += pr;
#pragma unroll
      for (int v = 0; v < DV; ++v) acc[v] = fmaf(pr, ld_f32(V + row + lane + 32 * v), acc[v]);
    }
    m = mn;
  }
  T* O = static_cast<T*>(p.out) + (int64_t)tok * p.o_st_tok + (int64_t)h * p.o_st_head;
  const float inv = 1.f / l;
#pragma unroll
  for (int v = 0; v < DV; ++v) st_from_f32(O + lane + 32 * v, acc[v] * inv);
}

template <typename T>
cudaError_t launch_t(const Params& p, cudaStream_t stream) {
  const int64_t inst = (int64_t)p.T * p.Hq;
  const unsigned grid = (unsigned)((inst + 3) / 4);
  if (p.D == 128)
    k7_baseline<T, 128><<<grid, 128, 0, stream>>>(p);
  else if (p.D == 64)
    k7_baseline<T, 64><<<grid, 128, 0, stream>>>(p);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_baseline(const Params& p, cudaStream_t stream) {
  if (p.T == 0) return cudaSuccess;
  if (p.dtype == 2) return launch_t<__half>(p, stream);
  return p.dtype == 1 ? launch_t<__nv_bfloat16>(p, stream) : launch_t<float>(p, stream);
}

}  // namespace pattn
