// K3 -- segment reduction of the parallel tiled softmax (§4.5, P:383-386;
// App. C).
//
// For a decode sequence split into n_b > 1 segments, K2 stored per segment s and
// query head h the unnormalised partial (m_s, l_s, acc_s) with m in the log2 domain
// (m = max_t scale*log2(e)*s_t).  The merge rescales "in a manner analogous to the
// iterative tiled softmax":
//     M = max_s m_s ;  w_s = 2^{m_s - M} (0 for an empty segment, m_s = -inf)
//     out[h][:] = sum_s w_s acc_s[:] / sum_s w_s l_s
// Segments are combined in index order (deterministic; no atomics).
// Grid: (num_seqs, Hkv * HG, D / 32); each 64-thread CTA handles 32 head-dim lanes of the
// <= 8 query heads of one (sequence, KV head, head group); non-decode or unsplit sequences
// exit at once.
#include "common.cuh"
#include "kernels.h"

namespace pattn {
namespace {

template <int D>
__global__ void __launch_bounds__(64) k3_reduce(Params p) {
  const int b = blockIdx.x;
  const int qb = p.cu_seqlens_q[b + 1] - p.cu_seqlens_q[b];
  if (!(p.decode_to_k2 && qb == 1)) return;
  const int c0 = p.cu_ch[b];
  const int n = p.cu_ch[b + 1] - c0;
  if (n <= 1) return;  // K2 wrote the final output itself
  const int kvh = blockIdx.y / p.HG, hg = blockIdx.y % p.HG;
  const int g_eff = min(8, p.G - hg * 8);
  const int head0 = kvh * p.G + hg * 8;
  const int tok = p.cu_seqlens_q[b];
  __nv_bfloat16* O = static_cast<__nv_bfloat16*>(p.out);
  for (int idx = threadIdx.x; idx < g_eff * 8; idx += blockDim.x) {
    const int h = head0 + idx / 8;
    const int d4 = blockIdx.z * 8 + idx % 8;
    float M = -INFINITY;
    for (int c = 0; c < n; ++c) M = fmaxf(M, p.part_m[(int64_t)(c0 + c) * p.Hq + h]);
    float den = 0.f;
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = 0; c < n; ++c) {
      const int64_t row = (int64_t)(c0 + c) * p.Hq + h;
      const float mc = p.part_m[row];
      const float w = (mc == -INFINITY) ? 0.f : exp2f(mc - M);
      den = fmaf(w, p.part_l[row], den);
      const float4 a = reinterpret_cast<const float4*>(p.part_acc + row * D)[d4];
      num.x = fmaf(w, a.x, num.x);
      num.y = fmaf(w, a.y, num.y);
      num.z = fmaf(w, a.z, num.z);
      num.w = fmaf(w, a.w, num.w);
    }
    const float inv = 1.f / den;
    uint2 packed;
    packed.x = pack_bf16(num.x * inv, num.y * inv);
    packed.y = pack_bf16(num.z * inv, num.w * inv);
    *reinterpret_cast<uint2*>(O + (int64_t)tok * p.o_st_tok + (int64_t)h * p.o_st_head + d4 * 4) = packed;
  }
}

}  // namespace

cudaError_t launch_reduce(const Params& p, cudaStream_t stream) {
  dim3 grid(p.B, p.Hkv * p.HG, p.D / 32);
  if (p.D == 64)
    k3_reduce<64><<<grid, 64, 0, stream>>>(p);
  else if (p.D == 128)
    k3_reduce<128><<<grid, 64, 0, stream>>>(p);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace pattn
