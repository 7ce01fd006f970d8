// K3 -- segment reduction of the parallel tiled softmax (§4.5, P:383-386;
// App. C).
//
// For a decode sequence split into n_b > 1 segments, K2 stored per segment s and
// query head h the unnormalised partial (m_s, l_s, acc_s) with m in the log2 domain
// (m = max_t scale*log2(e)*s_t).  The merge rescales "in a manner analogous to the
// iterative tiled softmax":
//     M = max_s m_s ;  w_s = 2^{m_s - M} (0 for an empty segment, m_s = -inf)
//     out[h][:] = sum_s w_s acc_s[:] / sum_s w_s l_s
// Segments are combined in a fixed order (deterministic; no atomics).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace pattn {
namespace {

// One (sequence, query head) item per W warps of a 256-thread CTA (8 / W items per CTA; W = 1
// for the usual few-segment case, W = 8 for long contexts or forced splitting).  Pass 1: the
// lanes read the segments' m_s 32 at a time, M = warp max (and, W > 1, CTA max).  Pass 2:
// segment c goes to warp c mod W of the item, whose lanes cover the D columns (D/32 each,
// coalesced 512 B per segment row at D = 128); the loop is unrolled so several segments'
// loads are in flight per warp (the round-1 version walked the segments one dependent load at a
// time per thread).  W > 1: the warps' (num, den) are combined through shared memory in warp
// order.  Fixed summation order for a given segment count and W: bitwise reproducible.
// Persistent grid (static launch grid): CTAs stride over the items; sequences that
// are not split decodes cost one check, so a padded CUDA-graph bucket pays almost nothing.
template <typename T, int D, int W>
__global__ void __launch_bounds__(256) k3_reduce(Params p) {
  constexpr int kCols = D / 32;   // columns per lane
  constexpr int kPerCta = 8 / W;  // items per CTA
  __shared__ float s_num[W > 1 ? 8 : 1][W > 1 ? D : 1];
  __shared__ float s_red[8][2];
  pdl_wait();  // the decode kernel's partials are complete and visible
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = warp / W, wi = warp % W;  // item slot in the CTA, warp within the item
  const int n_items = p.B * p.Hq;
  for (int base = blockIdx.x * kPerCta; base < n_items; base += gridDim.x * kPerCta) {
    const int item = base + sub;
    int n = 0, c0 = 0, b = 0, h = 0;
    if (item < n_items) {
      b = item / p.Hq;
      h = item - b * p.Hq;
      // the four metadata words in one round of loads (cu_ch counts 0 segments for non-decodes)
      const int q0 = p.cu_seqlens_q[b], q1 = p.cu_seqlens_q[b + 1];
      const int ch0 = p.cu_ch[b], ch1 = p.cu_ch[b + 1];
      if (p.decode_split && q1 - q0 == 1) {
        c0 = ch0;
        n = ch1 - ch0;
      }
    }
    const bool work = n > 1;  // n <= 1: the decode kernel wrote the final output itself
    // 1. M = max_s m_s
    float M = -INFINITY;
    if (work)
      for (int c = wi * 32 + lane; c < n; c += 32 * W) M = fmaxf(M, p.part_m[(int64_t)(c0 + c) * p.Hq + h]);
    M = warp_max(M);
    if (W > 1) {
      if (lane == 0) s_red[warp][0] = M;
      __syncthreads();
#pragma unroll
      for (int i = 0; i < W; ++i) M = fmaxf(M, s_red[sub * W + i][0]);
    }
    // 2. w_s = 2^{m_s - M} (0 for an empty segment); num = sum w_s acc_s, den = sum w_s l_s
    float num[kCols], den = 0.f;
#pragma unroll
    for (int k = 0; k < kCols; ++k) num[k] = 0.f;
    if (work) {
#pragma unroll 4
      for (int c = wi; c < n; c += W) {
        const int64_t row = (int64_t)(c0 + c) * p.Hq + h;
        const float mc = p.part_m[row];
        const float w = (mc == -INFINITY) ? 0.f : exp2f(mc - M);
        den = fmaf(w, p.part_l[row], den);
        const float* a = p.part_acc + row * D + lane * kCols;
        if constexpr (kCols == 4) {
          const float4 v = *reinterpret_cast<const float4*>(a);
          num[0] = fmaf(w, v.x, num[0]);
          num[1] = fmaf(w, v.y, num[1]);
          num[2] = fmaf(w, v.z, num[2]);
          num[3] = fmaf(w, v.w, num[3]);
        } else {
          const float2 v = *reinterpret_cast<const float2*>(a);
          num[0] = fmaf(w, v.x, num[0]);
          num[1] = fmaf(w, v.y, num[1]);
        }
      }
    }
    if (W > 1) {
#pragma unroll
      for (int k = 0; k < kCols; ++k) s_num[warp][lane * kCols + k] = num[k];
      if (lane == 0) s_red[warp][1] = den;
      __syncthreads();
      if (wi == 0) {
        for (int i = 1; i < W; ++i) {
#pragma unroll
          for (int k = 0; k < kCols; ++k) num[k] += s_num[warp + i][lane * kCols + k];
          den += s_red[warp + i][1];
        }
      }
    }
    if (work && wi == 0) {
      const float inv = 1.f / den;
      T* O = static_cast<T*>(p.out) + (int64_t)p.cu_seqlens_q[b] * p.o_st_tok + (int64_t)h * p.o_st_head +
             lane * kCols;
      if constexpr (sizeof(T) == 2) {
        if constexpr (kCols == 4) {
          uint2 packed;
          packed.x = pack2<T>(num[0] * inv, num[1] * inv);
          packed.y = pack2<T>(num[2] * inv, num[3] * inv);
          *reinterpret_cast<uint2*>(O) = packed;
        } else {
          *reinterpret_cast<uint32_t*>(O) = pack2<T>(num[0] * inv, num[1] * inv);
        }
      } else {
        if constexpr (kCols == 4)
          *reinterpret_cast<float4*>(O) = make_float4(num[0] * inv, num[1] * inv, num[2] * inv, num[3] * inv);
        else
          *reinterpret_cast<float2*>(O) = make_float2(num[0] * inv, num[1] * inv);
      }
    }
    if (W > 1) __syncthreads();  // shared partials are reused by the CTA's next items
  }
}

}  // namespace

template <typename T, int W>
cudaError_t launch_reduce_w(const Params& p, int grid, cudaStream_t stream) {
  if (p.D == 64) return launch_pdl(k3_reduce<T, 64, W>, dim3(grid), dim3(256), 0, stream, p);
  if (p.D == 128) return launch_pdl(k3_reduce<T, 128, W>, dim3(grid), dim3(256), 0, stream, p);
  return cudaErrorInvalidValue;
}

// Eight warps per item when sequences may have many segments (long contexts: max_seq_len hint
// > 16384, or forced splitting), else one warp per item.
template <typename T>
cudaError_t launch_reduce_t(const Params& p, cudaStream_t stream) {
  const bool many = p.max_seq_len_hint > 16384 || p.split_mode == 2;
  const int per_cta = many ? 1 : 8;
  const long long ctas = ((long long)p.B * p.Hq + per_cta - 1) / per_cta;
  const int grid = (int)std::max<long long>(1, std::min<long long>(ctas, (long long)p.num_sms * 8));
  return many ? launch_reduce_w<T, 8>(p, grid, stream) : launch_reduce_w<T, 1>(p, grid, stream);
}

cudaError_t launch_reduce(const Params& p, cudaStream_t stream) {
  if (p.dtype == 0) return launch_reduce_t<float>(p, stream);
  return p.dtype == 2 ? launch_reduce_t<__half>(p, stream) : launch_reduce_t<__nv_bfloat16>(p, stream);
}

}  // namespace pattn
