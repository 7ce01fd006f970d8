// K2 -- split-KV decode kernel: the paper's "parallel tiled softmax" (§4.5,
// P:367-391; App. C) for decode Q blocks (BLOCK_Q = 1), bf16.
//
// Work item = (decode segment c, KV head, head group of <= 8 query heads).  K5 split
// every decode sequence into n_b contiguous, equal-length ranges of KV blocks
// (segments); a persistent grid (2 CTAs per SM) strides over the items (static launch
// grid).  The Q block is the G query heads sharing the KV head (GQA
// packing), so every K/V byte is read from HBM exactly once.
//
// Memory path (the kernel is HBM-bound, arithmetic intensity G flop/byte):
//   warp 0 (producer): walks the block table (one coalesced load per 32 sub-blocks,
//     broadcast by shuffle) and for every 16-key sub-block of a paged block issues TMA
//     tile loads (cp.async.bulk.tensor.4d, box {64 d, 1 head, 16 slots, 1 block},
//     128B swizzle) of K and V into an NST-stage shared-memory ring guarded by
//     mbarriers.  Sub-blocks wholly past the sequence end are never fetched.
//   warps 1..NCW (consumers): sub-block g (CTA-global counter) goes to warp g % NCW.
//     Scores S^T[16 keys x 8 heads] = K . Q^T and O^T[D x 8] += V^T . P^T use
//     mma.sync.m16n8k16 (bf16 in, fp32 accumulate) fed by ldmatrix(.trans) from the
//     swizzled ring -- tensor cores here cut the instruction count (G = 8 would need
//     ~9 FMA-pipe ops per loaded element on SIMT), not the byte count.  Online softmax
//     per head in the log2 domain; row max by 3 shuffles, the sum l is kept
//     per lane and reduced once per item.  P is rounded to bf16 for the PV product
//     (reading R12); l uses unrounded p.
//   end of item: the NCW warp states are merged through shared memory; a
//     single-segment sequence writes bf16 output directly (acc / l), otherwise the
//     partial (m, l, acc) goes to the workspace for K3.
// Slots at positions >= L_b of the last sub-block may hold anything (NaN): scores are
// masked by select and those V rows are zeroed in shared memory before use
// (reading R13).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "trace.cuh"

PATTN_CTA_TRACE_DEFINE(k2)
PATTN_EV_TRACE_DEFINE(k2)

namespace pattn {
namespace {

constexpr int kSub = 16;  // keys per ring stage (one mma M tile)
constexpr int kItemRing = 16;
#ifndef PATTN_K2_NP
#define PATTN_K2_NP 4  // measured: per-SM decode rate +8% on 36 SMs vs 2 producers
#endif
constexpr int kNP = PATTN_K2_NP;  // producer warps
constexpr size_t kItemRingBytes = kItemRing * (2 * sizeof(uint64_t) + sizeof(int));

template <int D>
struct DecodeShape {
  static constexpr int kHalves = D / 64;  // 128-byte (64 x bf16) swizzle atoms per row
  static constexpr int kKC = D / 16;      // k-chunks of the QK^T mma / m-tiles of the PV mma
  static constexpr int kHalfBytes = kSub * 128;
  static constexpr int kOpBytes = kHalves * kHalfBytes;  // K (or V) of one 16-key sub-block
  static constexpr int kStageBytes = 2 * kOpBytes;
};

struct Item {
  int b, c, kvh, hg, sb0, sb1, nseg, L, tok;
};

// Segment c of decode sequence b covers paged blocks [kb0, kb1) (K5's plan), i.e. 16-key
// sub-blocks [kb0*bs/16, min(kb1*bs/16, ceil(L/16))).
__device__ __forceinline__ Item decode_item(const Params& p, int it) {
  Item x;
  const int units = p.Hkv * p.HG;
  x.c = it / units;
  const int u = it - x.c * units;
  x.kvh = u / p.HG;
  x.hg = u - x.kvh * p.HG;
  x.b = upper_bound_minus1(p.cu_ch, p.B, x.c);
  const int c0 = __ldg(p.cu_ch + x.b);
  x.nseg = __ldg(p.cu_ch + x.b + 1) - c0;
  x.L = __ldg(p.seq_lens + x.b);
  x.tok = __ldg(p.cu_seqlens_q + x.b);
  const int nblk = (x.L + p.bs - 1) / p.bs;
  const int per = (nblk + x.nseg - 1) / x.nseg;
  const int kb0 = (x.c - c0) * per;
  const int kb1 = min(nblk, kb0 + per);
  const int n16 = p.bs / kSub;
  x.sb0 = kb0 * n16;
  x.sb1 = min(kb1 * n16, (x.L + kSub - 1) / kSub);
  return x;
}

template <int D, int NCW, typename E>
__global__ void __launch_bounds__((NCW + kNP) * 32, 1)
    k2_decode(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Params p,
              int nst) {
  using S = DecodeShape<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nst * S::kStageBytes);
  uint64_t* empty = full + nst;
  float* scratch = reinterpret_cast<float*>(empty + nst);  // [NCW][16 + 8*D]
  constexpr int kScr = 16 + 8 * D;
  // dynamic work queue: the producer claims items from a global counter (reset by K5) and
  // publishes them to the consumer warps through a kItemRing-deep ring
  uint64_t* item_full = reinterpret_cast<uint64_t*>(scratch + NCW * kScr);
  uint64_t* item_empty = item_full + kItemRing;
  volatile int* item_ring = reinterpret_cast<volatile int*>(item_empty + kItemRing);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PATTN_CTA_BEGIN(k2);
  pdl_wait();  // K5's metadata (or, serial, the previous kernel's work) is complete and visible
  if (p.partition) {
    // two-stream SM partition: K5's P SMs belong to the prefill kernel K1 while it
    // still has Q blocks to claim -- a decode CTA placed there first (graph replays launch the
    // two branches in either order) leaves at once.  CTA 0 always works (progress guarantee).
    __shared__ int s_leave;
    if (threadIdx.x == 0) {
      const int pre_left = *reinterpret_cast<volatile int*>(p.hdr + kHdrPrefillCounter) <
                           p.hdr[kHdrTotalQBlocks] * p.Hkv;
      s_leave = blockIdx.x != 0 && partition_prefill_sm(sm_id(), p.hdr[kHdrPrefillCtas], p.num_sms) && pre_left;
    }
    __syncthreads();
    if (s_leave) return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < kItemRing; ++i) {
      mbar_init(&item_full[i], 1);
      mbar_init(&item_empty[i], NCW + kNP - 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  const int n_items = p.hdr[kHdrTotalChunks] * p.Hkv * p.HG;
  const int n16 = p.bs / kSub;

  if (warp == 0 || warp > NCW) {
    // ------------------------------------------------------------ producers
    // kNP producer warps (warp 0 and warp NCW+1): sub-block g of the CTA is issued by
    // producer g % kNP (the issue of a TMA box costs the issuing thread a few hundred
    // cycles, so one thread alone caps a CTA at ~14 B/clk).  Producer 0 claims the items.
    const int pw = warp == 0 ? 0 : warp - NCW;
    if (lane == 0) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
    }
    const uint64_t policy = l2_policy_evict_first();  // K/V are streamed exactly once
    uint32_t g = 0;  // CTA-global sub-block counter; a multiple of NCW (and kNP) at item start
    for (uint32_t ni = 0;; ++ni) {
      int it = 0;
      if (lane == 0) {
        const uint32_t slot = ni % kItemRing;
        if (pw == 0) {
          mbar_wait(&item_empty[slot], ((ni / kItemRing) & 1u) ^ 1u);
          it = atomicAdd(p.hdr + kHdrDecodeCounter, 1);
          item_ring[slot] = it;
          mbar_arrive(&item_full[slot]);
        } else {
          mbar_wait(&item_full[slot], (ni / kItemRing) & 1u);
          it = item_ring[slot];
          mbar_arrive(&item_empty[slot]);
        }
      }
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= n_items) {
        if (pw == 0 && lane == 0) {
          pdl_trigger();                              // no more items here: K3 may be scheduled
          atomicExch(p.hdr + kHdrDecodeClaimed, 1);  // and K1's late CTAs may take decode SMs
        }
        break;
      }
      const Item x = decode_item(p, it);
      const int32_t* bt = p.block_table + (int64_t)x.b * p.bt_stride;
      for (int j0 = x.sb0; j0 < x.sb1; j0 += 32) {
        const int n = min(32, x.sb1 - j0);
        const int id = lane < n ? __ldg(bt + (j0 + lane) / n16) : 0;
        for (int jj = pw; jj < n; jj += kNP) {
          const int blk = __shfl_sync(0xffffffffu, id, jj);
          const int slot0 = ((j0 + jj) % n16) * kSub;
          if (lane == 0) {
            const uint32_t gg = g + (uint32_t)(j0 - x.sb0 + jj);
            const uint32_t s = gg % nst;
            mbar_wait_tag(&empty[s], ((gg / nst) & 1u) ^ 1u, 1000000 + (int)gg, it, 0);
            PATTN_EV(k2, 0, gg);
            mbar_arrive_expect_tx(&full[s], S::kStageBytes);
            uint8_t* st = ring + (size_t)s * S::kStageBytes;
            // one box per operand: {64 d, 16 slots, D/64 d-halves} -> [half][slot][64 d]
            tma_load_5d_hint(st, &tmK, &full[s], 0, slot0, 0, x.kvh, blk, policy);
            tma_load_5d_hint(st + S::kOpBytes, &tmV, &full[s], 0, slot0, 0, x.kvh, blk, policy);
          }
        }
      }
      g += (uint32_t)(x.sb1 - x.sb0);
      // pad to a multiple of NCW with empty stages, so that every item starts on consumer
      // warp 0: sub-block j of an item always goes to warp j % NCW and the NCW-way merge
      // is bitwise independent of which CTA (and after which items) runs the item
      for (; g % NCW != 0; ++g) {
        if (lane == 0 && (int)(g % kNP) == pw) {
          const uint32_t s = g % nst;
          mbar_wait(&empty[s], ((g / nst) & 1u) ^ 1u);
          mbar_arrive(&full[s]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int cw = warp - 1;
  const int r = lane >> 2, c = lane & 3;       // mma fragment coordinates
  const int mat = lane >> 3, mrow = lane & 7;  // ldmatrix source coordinates
  float* scr = scratch + cw * kScr;
  using ET = typename E::T;
  ET* O = static_cast<ET*>(p.out);
  const ET* Q = static_cast<const ET*>(p.q);
  const uint32_t ring_u32 = smem_u32(ring);
  uint32_t g = 0;

  uint32_t ni = 0;
  for (;; ++ni) {
    const uint32_t slot = ni % kItemRing;
    mbar_wait(&item_full[slot], (ni / kItemRing) & 1u);
    const int it = item_ring[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&item_empty[slot]);
    if (it >= n_items) break;
    if (lane == 0 && cw == 0) PATTN_EV(k2, 4, ni);
    const Item x = decode_item(p, it);
    const int g_eff = min(8, p.G - x.hg * 8);
    const int head0 = x.kvh * p.G + x.hg * 8;

    // Q^T as the B operand of S^T = K . Q^T: b0 = Q[head r][16kc + 2c .. +1], b1 = +8
    uint32_t bq[S::kKC][2];
    {
      const ET* qrow = Q + (int64_t)x.tok * p.q_st_tok + (int64_t)(head0 + r) * p.q_st_head;
#pragma unroll
      for (int kc = 0; kc < S::kKC; ++kc) {
        bq[kc][0] = r < g_eff ? __ldg(reinterpret_cast<const uint32_t*>(qrow + kc * 16 + 2 * c)) : 0u;
        bq[kc][1] = r < g_eff ? __ldg(reinterpret_cast<const uint32_t*>(qrow + kc * 16 + 2 * c + 8)) : 0u;
      }
    }

    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float acc[S::kKC][4];
#pragma unroll
    for (int t = 0; t < S::kKC; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;

    const int nsb = x.sb1 - x.sb0;
    // Sub-block g (CTA-global counter) goes to consumer warp g % NCW, and nst is a multiple
    // of NCW, so every ring stage is always consumed by the same warp, in order.  (TMA loads
    // complete out of order: a waiter must have observed phase u-1 of a stage before it
    // waits on phase u, otherwise the parity test aliases and returns early.)  Items start
    // at g % NCW == 0 (the producer pads with empty stages), so warp cw takes j = cw mod NCW.
    // This warp's ring position, kept incrementally (one division per item instead of one per
    // stage: nst is a runtime value; it is a multiple of NCW, so stepping by NCW wraps cleanly).
    uint32_t ws = (g + cw) % nst, wph = ((g + cw) / nst) & 1u;
    // S^T[16 keys x 8 heads] = K . Q^T of sub-block jj (waits for its stage sq, phase sph)
    auto scores = [&](int jj, uint32_t sq, uint32_t sph, float (&sc)[4]) {
      const uint32_t gq = g + jj;
      if (lane == 0) PATTN_EV(k2, 1, gq);
      mbar_wait_tag(&full[sq], sph, (int)gq, it, jj);
      if (lane == 0) PATTN_EV(k2, 2, gq);
      const uint32_t kq = ring_u32 + sq * S::kStageBytes;
      sc[0] = sc[1] = sc[2] = sc[3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < S::kKC; ++kc) {
        const int key = (mat & 1) * 8 + mrow;
        const int dd = kc * 16 + (mat >> 1) * 8;
        const uint32_t addr = kq + (dd >> 6) * S::kHalfBytes + key * 128 + ((((dd & 63) >> 3) ^ (key & 7)) << 4);
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4(addr, a0, a1, a2, a3);
        E::mma(sc, a0, a1, a2, a3, bq[kc][0], bq[kc][1]);
      }
    };
    for (int j = cw; j < nsb; j += NCW) {
      const uint32_t gg = g + j;
      const uint32_t s = ws;
      float sc[4];
      scores(j, ws, wph, sc);
      ws += NCW;
      if (ws >= (uint32_t)nst) ws -= (uint32_t)nst, wph ^= 1u;
      const uint32_t kst = ring_u32 + s * S::kStageBytes;
      const uint32_t vst = kst + S::kOpBytes;
      const int valid = x.L - (x.sb0 + j) * kSub;  // slots [0, valid) hold real keys
      if (valid < kSub) {
        // zero V rows past the sequence end (they may hold NaN; 0 * NaN = NaN in the mma)
        uint8_t* vgen = ring + (size_t)s * S::kStageBytes + S::kOpBytes;
        const int nrow = kSub - valid;
        for (int e = lane; e < nrow * 8 * S::kHalves; e += 32) {
          const int h = e / (nrow * 8);
          const int rem = e - h * nrow * 8;
          const int row = valid + rem / 8;
          const int ch = rem & 7;
          *reinterpret_cast<uint4*>(vgen + h * S::kHalfBytes + row * 128 + ch * 16) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
      }
      // sc[0..1]: key r, heads 2c, 2c+1; sc[2..3]: key r + 8
      const float s0 = r < valid ? sc[0] * p.scale_log2 : -INFINITY;
      const float s1 = r < valid ? sc[1] * p.scale_log2 : -INFINITY;
      const float s2 = r + 8 < valid ? sc[2] * p.scale_log2 : -INFINITY;
      const float s3 = r + 8 < valid ? sc[3] * p.scale_log2 : -INFINITY;
      float mt0 = fmaxf(s0, s2), mt1 = fmaxf(s1, s3);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        mt0 = fmaxf(mt0, __shfl_xor_sync(0xffffffffu, mt0, o));
        mt1 = fmaxf(mt1, __shfl_xor_sync(0xffffffffu, mt1, o));
      }
      const float mn0 = fmaxf(m0, mt0), mn1 = fmaxf(m1, mt1);  // finite: every sub-block has a valid key
      const float al0 = fast_exp2(m0 - mn0), al1 = fast_exp2(m1 - mn1);
      const float p0 = fast_exp2(s0 - mn0), p1 = fast_exp2(s1 - mn1);
      const float p2 = fast_exp2(s2 - mn0), p3 = fast_exp2(s3 - mn1);
      l0 = fmaf(l0, al0, p0 + p2);
      l1 = fmaf(l1, al1, p1 + p3);
      m0 = mn0;
      m1 = mn1;
#pragma unroll
      for (int t = 0; t < S::kKC; ++t) {
        acc[t][0] *= al0;
        acc[t][1] *= al1;
        acc[t][2] *= al0;
        acc[t][3] *= al1;
      }
      // P^T as the B operand of O^T = V^T . P^T (transpose the 8x8 halves in registers)
      const uint32_t pb0 = movmatrix_trans(E::pack(p0, p1));
      const uint32_t pb1 = movmatrix_trans(E::pack(p2, p3));
#pragma unroll
      for (int t = 0; t < S::kKC; ++t) {
        const int key = (mat >> 1) * 8 + mrow;
        const int dd = t * 16 + (mat & 1) * 8;
        const uint32_t addr = vst + (dd >> 6) * S::kHalfBytes + key * 128 + ((((dd & 63) >> 3) ^ (key & 7)) << 4);
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4_trans(addr, a0, a1, a2, a3);
        E::mma(acc[t], a0, a1, a2, a3, pb0, pb1);
      }
      __syncwarp();
      if (valid < kSub) fence_proxy_async_smem();  // generic zero-writes before the next TMA fill
      if (lane == 0) mbar_arrive(&empty[s]);
      if (lane == 0) PATTN_EV(k2, 3, gg);
    }
    g += nsb;
    for (; g % NCW != 0; ++g) {  // the producer's padding stages
      if ((int)(g % NCW) == cw) {
        const uint32_t s = g % nst;
        mbar_wait(&full[s], (g / nst) & 1u);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }

    // ---- merge the NCW warp states of this item
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, o);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    if (r == 0) {
      scr[2 * c] = m0;
      scr[2 * c + 1] = m1;
      scr[8 + 2 * c] = l0;
      scr[8 + 2 * c + 1] = l1;
    }
#pragma unroll
    for (int t = 0; t < S::kKC; ++t) {
      scr[16 + (2 * c) * D + 16 * t + r] = acc[t][0];
      scr[16 + (2 * c + 1) * D + 16 * t + r] = acc[t][1];
      scr[16 + (2 * c) * D + 16 * t + r + 8] = acc[t][2];
      scr[16 + (2 * c + 1) * D + 16 * t + r + 8] = acc[t][3];
    }
    named_bar_sync(1, NCW * 32);
    const int ct = threadIdx.x - 32;
    for (int idx = ct; idx < g_eff * D; idx += NCW * 32) {
      const int h = idx / D, d = idx - h * D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NCW; ++w) M = fmaxf(M, scratch[w * kScr + h]);
      float num = 0.f, den = 0.f;
#pragma unroll
      for (int w = 0; w < NCW; ++w) {
        const float mw = scratch[w * kScr + h];
        const float wt = mw == -INFINITY ? 0.f : fast_exp2(mw - M);
        num = fmaf(wt, scratch[w * kScr + 16 + h * D + d], num);
        den = fmaf(wt, scratch[w * kScr + 8 + h], den);
      }
      if (x.nseg == 1) {
        O[(int64_t)x.tok * p.o_st_tok + (int64_t)(head0 + h) * p.o_st_head + d] = from_f32<ET>(num / den);
      } else {
        const int64_t row = (int64_t)x.c * p.Hq + head0 + h;
        p.part_acc[row * D + d] = num;
        if (d == 0) {
          p.part_m[row] = M;
          p.part_l[row] = den;
        }
      }
    }
    named_bar_sync(1, NCW * 32);
    if (lane == 0 && cw == 0) PATTN_EV(k2, 5, ni);
  }
  if (warp == 1 && lane == 0) PATTN_CTA_END(k2, ni);
}

int env_or(const char* name, int dflt);

template <int D, int NCW, typename E>
cudaError_t launch_dw(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK, const CUtensorMap& tmV,
                      cudaStream_t stream) {
  auto kern = k2_decode<D, NCW, E>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), dl.smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3(dl.grid), dim3((NCW + kNP) * 32), dl.smem, stream, tmK, tmV, p, dl.stages);
}

template <int D>
cudaError_t launch_d(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK, const CUtensorMap& tmV,
                     cudaStream_t stream) {
  if (p.dtype == 2) {
    if (dl.consumer_warps == 8) return launch_dw<D, 8, EltF16>(p, dl, tmK, tmV, stream);
    return launch_dw<D, 4, EltF16>(p, dl, tmK, tmV, stream);
  }
  if (dl.consumer_warps == 8) return launch_dw<D, 8, EltBf16>(p, dl, tmK, tmV, stream);
  return launch_dw<D, 4, EltBf16>(p, dl, tmK, tmV, stream);
}

int env_or(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

}  // namespace

// Launch shape: one or two CTAs per SM, each with 1 producer + NCW consumer warps and an
// NST-stage ring; ~160 KB of K/V in flight per SM.  Env overrides for sweeps:
// PATTN_DECODE_WARPS (4|8), PATTN_DECODE_CTAS (1|2), PATTN_DECODE_RING_KB.
DecodeLaunch plan_decode(const Params& p, int num_sms, size_t max_smem, int ctas_per_sm) {
  DecodeLaunch dl;
  dl.consumer_warps = env_or("PATTN_DECODE_WARPS", 4) == 8 ? 8 : 4;
  int ctas = ctas_per_sm;  // tuning tree / PATTN_DECODE_CTAS, resolved by the planner
  if (ctas < 1) ctas = 1;
  if (ctas > 4) ctas = 4;
  const size_t stage = (size_t)4 * kSub * p.D;  // K + V of one 16-key sub-block, bf16
  const size_t scratch = (size_t)dl.consumer_warps * (16 + 8 * p.D) * sizeof(float);
  const size_t fixed = 1024 /*align slack*/ + scratch + kItemRingBytes;
  const size_t per_cta = (max_smem < 228 * 1024 ? max_smem : 228 * 1024) / ctas - 1024;
  const size_t budget = per_cta > fixed ? per_cta - fixed : 0;
  size_t want = (size_t)env_or("PATTN_DECODE_RING_KB", 96) * 1024;
  if (want > budget) want = budget;
  int st = (int)(want / (stage + 16));
  if (st > 64) st = 64;
  st -= st % dl.consumer_warps;  // stage s is always consumed by warp s % NCW (see kernel)
  if (st < dl.consumer_warps) st = dl.consumer_warps;
  dl.stages = st;
  dl.smem = fixed + (size_t)st * (stage + 16);
  const long long max_items = (long long)p.max_chunks * p.Hkv * p.HG;
  const long long g = (long long)std::min(num_sms, std::max(1, env_or("PATTN_DECODE_SMS", num_sms))) * ctas;
  dl.grid = (int)(max_items < g ? max_items : g);
  if (dl.grid < 1) dl.grid = 1;
  return dl;
}

cudaError_t launch_decode(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK, const CUtensorMap& tmV,
                          cudaStream_t stream) {
  if (p.D == 128) return launch_d<128>(p, dl, tmK, tmV, stream);
  if (p.D == 64) return launch_d<64>(p, dl, tmK, tmV, stream);
  return cudaErrorInvalidValue;
}

}  // namespace pattn
