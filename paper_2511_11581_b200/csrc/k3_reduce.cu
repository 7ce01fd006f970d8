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
// Grid: (num_seqs, Hkv * HG, D / 32); each CTA handles 32 head-dim lanes of the <= 8 query
// heads of one (sequence, KV head, head group); non-decode or unsplit sequences exit at once.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace pattn {
namespace {

// 64 x kMaxGroups threads = segment groups x 8 heads x 8 float4 columns: thread (sg, h, d4)
// reduces the segments s = sg (mod SG) of head h for columns 4*d4 .. 4*d4+3 of the item's
// 32-column slice, then the groups are combined through shared memory in group order
// (deterministic).  The number of active groups SG = clamp(ceil(n / 8), 1, kMaxGroups) follows
// the sequence's actual segment count n (config 2: 5 segments -> 1 group; config 4: 37 -> 4);
// for a given n and launch variant the order of the additions is fixed (bitwise reproducible).
// Persistent grid (static launch grid): CTAs stride over the (sequence, KV head x
// head group, 32-column slice) items; sequences that are not split decodes cost one check, so
// a CUDA-graph bucket padded with empty sequences pays almost nothing for them.
template <typename T, int D, int kMaxGroups>
__global__ void __launch_bounds__(64 * kMaxGroups) k3_reduce(Params p) {
  __shared__ float s_max[kMaxGroups][8];
  __shared__ float4 s_num[kMaxGroups][8][8];
  __shared__ float s_den[kMaxGroups][8];
  pdl_wait();  // the decode kernel's partials are complete and visible
  const int ny = p.Hkv * p.HG, nz = D / 32;
  const int n_items = p.B * ny * nz;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int b = item / (ny * nz);
    const int yz = item - b * ny * nz;
    const int by = yz / nz, bz = yz - by * nz;
    const int qb = p.cu_seqlens_q[b + 1] - p.cu_seqlens_q[b];
    if (!(p.decode_split && qb == 1)) continue;
    const int c0 = p.cu_ch[b];
    const int n = p.cu_ch[b + 1] - c0;
    if (n <= 1) continue;  // the decode kernel wrote the final output itself
    const int groups = min(kMaxGroups, (n + 7) / 8);
    const int kvh = by / p.HG, hg = by % p.HG;
    const int g_eff = min(8, p.G - hg * 8);
    const int head0 = kvh * p.G + hg * 8;
    const int tok = p.cu_seqlens_q[b];
    const int d4 = threadIdx.x & 7, h = (threadIdx.x >> 3) & 7, sg = threadIdx.x >> 6;
    const bool active = h < g_eff && sg < groups;
    const int d4g = bz * 8 + d4;  // float4 column within the head
    // 1. M = max_s m_s per head (each group over its segments, then across groups)
    float M = -INFINITY;
    if (active)
      for (int c = sg; c < n; c += groups) M = fmaxf(M, p.part_m[(int64_t)(c0 + c) * p.Hq + head0 + h]);
    if (d4 == 0) s_max[sg][h] = M;
    __syncthreads();
    for (int g = 0; g < groups; ++g) M = fmaxf(M, s_max[g][h]);
    // 2. w_s = 2^{m_s - M} (0 for an empty segment); num = sum w_s acc_s, den = sum w_s l_s
    float den = 0.f;
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
    if (active) {
  #pragma unroll 8
      for (int c = sg; c < n; c += groups) {
        const int64_t row = (int64_t)(c0 + c) * p.Hq + head0 + h;
        const float mc = p.part_m[row];
        const float w = (mc == -INFINITY) ? 0.f : exp2f(mc - M);
        den = fmaf(w, p.part_l[row], den);
        const float4 a = reinterpret_cast<const float4*>(p.part_acc + row * D)[d4g];
        num.x = fmaf(w, a.x, num.x);
        num.y = fmaf(w, a.y, num.y);
        num.z = fmaf(w, a.z, num.z);
        num.w = fmaf(w, a.w, num.w);
      }
    }
    s_num[sg][h][d4] = num;
    if (d4 == 0) s_den[sg][h] = den;
    __syncthreads();
    if (sg == 0 && active) {
      float4 t = s_num[0][h][d4];
      float dd = s_den[0][h];
      for (int g = 1; g < groups; ++g) {
        const float4 u = s_num[g][h][d4];
        t.x += u.x;
        t.y += u.y;
        t.z += u.z;
        t.w += u.w;
        dd += s_den[g][h];
      }
      const float inv = 1.f / dd;
      T* O = static_cast<T*>(p.out) + (int64_t)tok * p.o_st_tok + (int64_t)(head0 + h) * p.o_st_head + d4g * 4;
      if constexpr (sizeof(T) == 2) {
        uint2 packed;
        packed.x = pack2<T>(t.x * inv, t.y * inv);
        packed.y = pack2<T>(t.z * inv, t.w * inv);
        *reinterpret_cast<uint2*>(O) = packed;
      } else {
        *reinterpret_cast<float4*>(O) = make_float4(t.x * inv, t.y * inv, t.z * inv, t.w * inv);
      }
    }
    __syncthreads();  // shared partials are reused by the CTA's next item
  }
}

}  // namespace

template <typename T, int G>
cudaError_t launch_reduce_g(const Params& p, int grid, cudaStream_t stream) {
  if (p.D == 64)
    return launch_pdl(k3_reduce<T, 64, G>, dim3(grid), dim3(64 * G), 0, stream, p);
  if (p.D == 128)
    return launch_pdl(k3_reduce<T, 128, G>, dim3(grid), dim3(64 * G), 0, stream, p);
  return cudaErrorInvalidValue;
}

// Up to 4 segment groups (256 threads) when sequences may have many segments: long contexts
// (max_seq_len hint > 16384) or forced splitting; the group count actually used follows each
// sequence's segment count.  Otherwise one group (64 threads, the common few-segment case).
template <typename T>
cudaError_t launch_reduce_t(const Params& p, cudaStream_t stream) {
  const long long items = (long long)p.B * p.Hkv * p.HG * (p.D / 32);
  const bool many = p.max_seq_len_hint > 16384 || p.split_mode == 2;
  const int grid = (int)std::min<long long>(items, (long long)p.num_sms * (many ? 8 : 16));
  return many ? launch_reduce_g<T, 4>(p, std::max(grid, 1), stream) : launch_reduce_g<T, 1>(p, std::max(grid, 1), stream);
}

cudaError_t launch_reduce(const Params& p, cudaStream_t stream) {
  if (p.dtype == 0) return launch_reduce_t<float>(p, stream);
  return p.dtype == 2 ? launch_reduce_t<__half>(p, stream) : launch_reduce_t<__nv_bfloat16>(p, stream);
}

}  // namespace pattn
