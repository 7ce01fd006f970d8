// K4 -- generic SIMT Q-block kernel (§4.4 Q-Block; App. B).
//
// The exact-ish path: fp32 inputs (tolerance 1e-5, no tf32) and the fallback for bf16
// shapes the specialised kernels do not cover (block sizes that are not a multiple of
// 16, head_dim 64 prefill).  One CTA (4 warps) processes one work item = (Q block,
// KV head): BLOCK_M = BLOCK_Q * G rows, token-major / head-minor (row r -> token
// r / G, head kvh*G + r % G; reading R8).  K/V tiles of 32 keys are gathered through
// the block table into shared memory ONCE per Q block and reused by all
// rows (the Q-block arithmetic-density argument); every row runs the
// online softmax of P:249-266 (m, l, acc in registers, division delayed to the end)
// with its own causal limit ctx + i + 1.
//
// Persistent grid (static launch grid): CTAs stride over the
// total_q_blocks * Hkv items produced by K5, last Q blocks first (longest first).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace pattn {
namespace {

constexpr int kWarps = 4;
constexpr int kTileKeys = 32;

template <typename T, int D, int RPW>
__global__ void __launch_bounds__(kWarps * 32) k4_generic(Params p) {
  extern __shared__ float smem[];
  constexpr int DV = D / 32;  // accumulator elements per lane
  const int G = p.G, BQ = p.block_q, BM = BQ * G;
  float* sQ = smem;                        // [BM][D]
  float* sK = sQ + BM * D;                 // [32][D+1]  (padded: lane-per-key reads conflict-free)
  float* sV = sK + kTileKeys * (D + 1);    // [32][D]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* __restrict__ Q = static_cast<const T*>(p.q);
  const T* __restrict__ K = static_cast<const T*>(p.k);
  const T* __restrict__ V = static_cast<const T*>(p.v);
  T* __restrict__ O = static_cast<T*>(p.out);

  pdl_wait();  // K5's metadata is complete and visible
  const int total_qb = p.hdr[kHdrTotalQBlocks];
  const int n_pre = total_qb * p.Hkv;
  // decode segments (split-KV) when the decode kernel K2 cannot take them: one item
  // per (segment, KV head) covering the G query heads of that KV head
  const int n_items = n_pre + (p.k4_decodes ? p.hdr[kHdrTotalChunks] * p.Hkv : 0);
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    int b, kvh, q0, ntok, tok0, ctx, kv_begin, kv_end, nseg = 1, chunk = 0;
    if (it < n_pre) {
      const int j = total_qb - 1 - it / p.Hkv;  // global Q-block id, last first
      kvh = it % p.Hkv;
      b = upper_bound_minus1(p.cu_qb, p.B, j);  // App. B P:46 binary search
      const int qblk = j - p.cu_qb[b];
      q0 = p.cu_seqlens_q[b];
      const int qlen = p.cu_seqlens_q[b + 1] - q0;
      ctx = p.seq_lens[b] - qlen;
      tok0 = qblk * BQ;
      ntok = min(BQ, qlen - tok0);
      kv_begin = 0;
      kv_end = ctx + tok0 + ntok;  // keys visible to the last row of the block
    } else {
      const int u = it - n_pre;
      chunk = u / p.Hkv;
      kvh = u - chunk * p.Hkv;
      b = upper_bound_minus1(p.cu_ch, p.B, chunk);
      const int c0 = p.cu_ch[b];
      nseg = p.cu_ch[b + 1] - c0;
      const int L = p.seq_lens[b];
      const int nblk = (L + p.bs - 1) / p.bs;
      const int per = (nblk + nseg - 1) / nseg;  // K5's equal block ranges (reading R9)
      const int kb0 = (chunk - c0) * per;
      q0 = p.cu_seqlens_q[b];
      ctx = L - 1;
      tok0 = 0;
      ntok = 1;
      kv_begin = min(kb0 * p.bs, L);
      kv_end = min((kb0 + per) * p.bs, L);
    }
    const int32_t* bt = p.block_table + (int64_t)b * p.bt_stride;

    __syncthreads();  // previous item finished with sQ
    for (int idx = threadIdx.x; idx < BM * D; idx += kWarps * 32) {
      int r = idx / D, d = idx - r * D;
      int tk = r / G;
      float x = 0.f;
      if (tk < ntok) {
        int h = kvh * G + (r - tk * G);
        x = to_f32(Q[(int64_t)(q0 + tok0 + tk) * p.q_st_tok + (int64_t)h * p.q_st_head + d]);
      }
      sQ[idx] = x;
    }

    float m[RPW], l[RPW], acc[RPW][DV];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      m[i] = -INFINITY;
      l[i] = 0.f;
#pragma unroll
      for (int k = 0; k < DV; ++k) acc[i][k] = 0.f;
    }

    for (int t0 = kv_begin; t0 < kv_end; t0 += kTileKeys) {
      __syncthreads();
      if (p.kv_vec16) {
        // 16-byte loads (8 bf16 / 4 fp32 per thread and operand): the tile's K and V rows are
        // contiguous head_dim vectors, so a warp reads whole 128-byte lines
        constexpr int kVec = 16 / (int)sizeof(T), kChunks = D / kVec;
#pragma unroll 2
        for (int idx = threadIdx.x; idx < kTileKeys * kChunks; idx += kWarps * 32) {
          const int jj = idx / kChunks, d = (idx - jj * kChunks) * kVec;
          const int t = t0 + jj;
          uint4 kr = make_uint4(0, 0, 0, 0), vr = make_uint4(0, 0, 0, 0);
          if (t < kv_end) {  // never touch slots past the visible range (may hold NaN, reading R13)
            const int64_t off = (int64_t)bt[t / p.bs] * p.kv_st_blk + (int64_t)(t % p.bs) * p.kv_st_tok +
                                (int64_t)kvh * p.kv_st_head + d;
            kr = __ldg(reinterpret_cast<const uint4*>(K + off));
            vr = __ldg(reinterpret_cast<const uint4*>(V + off));
          }
          const T* ke = reinterpret_cast<const T*>(&kr);
          const T* ve = reinterpret_cast<const T*>(&vr);
#pragma unroll
          for (int e = 0; e < kVec; ++e) {
            sK[jj * (D + 1) + d + e] = to_f32(ke[e]);
            sV[jj * D + d + e] = to_f32(ve[e]);
          }
        }
      } else {
        for (int idx = threadIdx.x; idx < kTileKeys * D; idx += kWarps * 32) {
          int jj = idx / D, d = idx - jj * D;
          int t = t0 + jj;
          float kx = 0.f, vx = 0.f;
          if (t < kv_end) {  // never touch slots past the visible range (may hold NaN, reading R13)
            int64_t off = (int64_t)bt[t / p.bs] * p.kv_st_blk + (int64_t)(t % p.bs) * p.kv_st_tok +
                          (int64_t)kvh * p.kv_st_head + d;
            kx = to_f32(K[off]);
            vx = to_f32(V[off]);
          }
          sK[jj * (D + 1) + d] = kx;
          sV[jj * D + d] = vx;
        }
      }
      __syncthreads();

#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const int r = warp + i * kWarps;
        if (r >= BM) break;
        const int tk = r / G;
        if (tk >= ntok) continue;
        const int row_end = min(ctx + tok0 + tk + 1, kv_end);  // keys 0 .. ctx+i (self-inclusive)
        if (t0 >= row_end) continue;              // warp-uniform
        const int t = t0 + lane;
        float s = -INFINITY;
        if (t < row_end) {
          const float* qr = sQ + r * D;
          const float* kr = sK + lane * (D + 1);
          float dot = 0.f;
#pragma unroll 16
          for (int d = 0; d < D; ++d) dot = fmaf(qr[d], kr[d], dot);
          s = dot * p.scale_log2;  // log2 domain: e^{x} = 2^{x log2 e}
        }
        const float m_new = fmaxf(m[i], warp_max(s));
        const float alpha = exp2f(m[i] - m_new);  // m = -inf -> 0
        const float pe = (t < row_end) ? exp2f(s - m_new) : 0.f;
        l[i] = l[i] * alpha + warp_sum(pe);
#pragma unroll
        for (int k = 0; k < DV; ++k) acc[i][k] *= alpha;
#pragma unroll 8
        for (int jj = 0; jj < kTileKeys; ++jj) {
          const float pj = __shfl_sync(0xffffffffu, pe, jj);
          const float* vr = sV + jj * D + lane;
#pragma unroll
          for (int k = 0; k < DV; ++k) acc[i][k] = fmaf(pj, vr[32 * k], acc[i][k]);
        }
        m[i] = m_new;
      }
    }

#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int r = warp + i * kWarps;
      if (r >= BM) break;
      const int tk = r / G;
      if (tk >= ntok) continue;
      const int h = kvh * G + (r - tk * G);
      if (nseg > 1) {
        // partial (m, l, acc) of this segment for K3; m in the log2 domain;
        // an empty segment leaves m = -inf, l = 0, acc = 0 (skipped by the merge)
        const int64_t row = (int64_t)chunk * p.Hq + h;
        if (lane == 0) {
          p.part_m[row] = m[i];
          p.part_l[row] = l[i];
        }
#pragma unroll
        for (int k = 0; k < DV; ++k) p.part_acc[row * D + lane + 32 * k] = acc[i][k];
        continue;
      }
      T* o = O + (int64_t)(q0 + tok0 + tk) * p.o_st_tok + (int64_t)h * p.o_st_head;
      const float inv = 1.f / l[i];
#pragma unroll
      for (int k = 0; k < DV; ++k) o[lane + 32 * k] = from_f32<T>(acc[i][k] * inv);
    }
  }
}

template <typename T, int D, int RPW>
cudaError_t launch_t(const Params& p, int grid, cudaStream_t stream) {
  size_t smem = generic_smem_bytes(p);
  auto kern = k4_generic<T, D, RPW>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3(grid), dim3(kWarps * 32), smem, stream, p);
}

template <typename T, int D>
cudaError_t launch_d(const Params& p, int grid, int rpw, cudaStream_t stream) {
  return rpw <= 8 ? launch_t<T, D, 8>(p, grid, stream) : launch_t<T, D, 16>(p, grid, stream);
}

}  // namespace

size_t generic_smem_bytes(const Params& p) {
  const int BM = p.block_q * p.G;
  return sizeof(float) * ((size_t)BM * p.D + (size_t)kTileKeys * (p.D + 1) + (size_t)kTileKeys * p.D);
}

cudaError_t launch_generic(const Params& p, int grid, int rows_per_warp, cudaStream_t stream) {
  if (p.dtype == 0) {
    if (p.D == 64) return launch_d<float, 64>(p, grid, rows_per_warp, stream);
    if (p.D == 128) return launch_d<float, 128>(p, grid, rows_per_warp, stream);
  } else {
    if (p.dtype == 2) {
      if (p.D == 64) return launch_d<__half, 64>(p, grid, rows_per_warp, stream);
      if (p.D == 128) return launch_d<__half, 128>(p, grid, rows_per_warp, stream);
    }
    if (p.D == 64) return launch_d<__nv_bfloat16, 64>(p, grid, rows_per_warp, stream);
    if (p.D == 128) return launch_d<__nv_bfloat16, 128>(p, grid, rows_per_warp, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace pattn
