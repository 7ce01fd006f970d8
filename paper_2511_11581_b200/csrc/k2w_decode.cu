// K2W -- split-KV decode with head-wide TMA boxes: the same computation as K2 (§4.5
// "parallel tiled softmax"; App. C; GQA packing P:344-350), reorganised
// around how many bytes ONE TMA request brings in.
//
// Measured on B200 (scripts/micro/kv_stream.cu, one CTA per SM, no consumers): an SM that
// streams 4 KB boxes (K2's unit: 16 keys of ONE KV head) tops out at ~26-28 GB/s per issuing
// thread and ~56 GB/s with K2's four producer warps, whatever the number of bytes in flight --
// the cost is per request.  A box of the same 5-D view that spans HB KV heads (32 KB at HB = 8,
// D = 128) reaches 137 GB/s/SM with 128 KB in flight and 167 GB/s/SM with 192 KB.  When the
// decode kernel owns only the SMs the prefill kernel leaves it (two-stream mixed batches), its
// per-SM rate decides the step, so K2W trades K2's per-head work items for head-group items:
//
//   work item = (decode segment c, group of HB KV heads); K5 plans segments with Hkv / HB
//     items per segment (units per segment, Params::decode_hb).
//   warp 0 (producer): per 16-key sub-block of the segment, ONE K box and ONE V box
//     {64 d, 16 slots, D/64 halves, HB heads, 1 block} into two consecutive entries of a ring
//     of single-operand entries (each lands as HB head-major copies of K2's [half][slot][64 d]
//     layout, 128B-swizzled).  Block sizes that are not a multiple of 16 (kGather): four
//     producer warps fill the same entries row by row with cp.async instead.
//   warps (consumers): warp w owns KV head hb*HB + w for the whole item -- every sub-block, in
//     key order -- with its G <= 8 query heads as the N = 8 columns of mma.sync (S^T = K.Q^T,
//     O^T = V^T.P^T, online softmax in the log2 domain with a lazy running max).  An entry is
//     released when all HB warps have consumed it: K(j) right after the scores, V(j) after PV.
//     No cross-warp merge: each warp writes its head's output (single-segment sequences) or
//     (m, l, acc) partial for K3 straight from its mma fragments.
// Requirements (planner): G <= 16 (one or two head groups of <= 8 query heads: one consumer warp
// per (KV head, head group)), HB in {2, 4, 8} dividing Hkv, 16-byte aligned
// K/V rows.  V rows past the segment's keys are zeroed in shared memory before PV (slots past
// the sequence end may hold NaN; reading R13), scores there are masked by select.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "trace.cuh"

PATTN_CTA_TRACE_DEFINE(k2w)

namespace pattn {
namespace {

constexpr int kSub = 16;       // keys per sub-block (one mma M tile)
constexpr int kItemRing = 8;   // producer -> consumers item queue
constexpr float kLazyMax = 8.f;  // log2 domain: rescale only when a score exceeds the running max by > 2^8

template <int D, int HB>
struct WideShape {
  static constexpr int kHalves = D / 64;
  static constexpr int kKC = D / 16;                     // k-chunks of S^T, m-tiles of O^T
  static constexpr int kHalfBytes = kSub * 128;          // [slot][64 d] of one d half
  static constexpr int kHeadBytes = kHalves * kHalfBytes;  // one head's 16 keys of K (or V)
  static constexpr int kOpBytes = HB * kHeadBytes;       // one box (ring entry): HB heads of K or of V
};

struct WItem {
  int b, c, hb, sb0, sb1, nseg, L, tok;
  int k0, k1;  // the segment's keys [k0, k1): sub-block j holds keys k0 + 16 j ..
};

// Segment c of decode sequence b covers paged blocks [kb0, kb1) of K5's plan (the same
// equal-split rule as K2, reading R9); hb selects the KV-head group.
__device__ __forceinline__ WItem wide_item(const Params& p, int it, int ngroups) {
  WItem x;
  x.c = it / ngroups;
  x.hb = it - x.c * ngroups;
  x.b = upper_bound_minus1(p.cu_ch, p.B, x.c);
  const int c0 = __ldg(p.cu_ch + x.b);
  x.nseg = __ldg(p.cu_ch + x.b + 1) - c0;
  x.L = __ldg(p.seq_lens + x.b);
  x.tok = __ldg(p.cu_seqlens_q + x.b);
  const int nblk = (x.L + p.bs - 1) / p.bs;
  const int per = (nblk + x.nseg - 1) / x.nseg;
  const int kb0 = (x.c - c0) * per;
  const int kb1 = min(nblk, kb0 + per);
  x.k0 = kb0 * p.bs;
  x.k1 = min(kb1 * p.bs, x.L);
  const int n16 = p.bs / kSub;  // TMA path (bs a multiple of 16): sub-blocks are page-aligned
  x.sb0 = kb0 * n16;
  x.sb1 = x.sb0 + (x.k1 - x.k0 + kSub - 1) / kSub;
  return x;
}

// kGather: block sizes that are not a multiple of 16 (no TMA box fits a page): four producer
// warps gather the same ring entries row by row with 16-byte cp.async (one block-table lookup per
// key row, any block size, 16-byte aligned rows), completing on the entry's mbarrier through
// cp.async.mbarrier.arrive.noinc; the consumers are unchanged.
// HGW: head groups of <= 8 query heads per KV head (G <= 8: 1; 8 < G <= 16: 2); the consumer
// warps are (KV head, head group) pairs.
template <int D, int HB, typename E, bool kGather, int HGW>
__global__ void __launch_bounds__((HB * HGW + (kGather ? 4 : 2)) * 32, 1)
    k2w_decode(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Params p,
               int nent) {
  using S = WideShape<D, HB>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // Ring of nent entries, each ONE operand box (K or V of a 16-key sub-block, HB heads): the
  // producer fills K(j), V(j) into consecutive entries; the consumers release K(j) right after
  // the scores, so the next boxes are in flight while PV(j) still reads V(j).
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)nent * S::kOpBytes);
  uint64_t* empty = full + nent;
  uint64_t* item_full = empty + nent;
  uint64_t* item_empty = item_full + kItemRing;
  volatile int* item_ring = reinterpret_cast<volatile int*>(item_empty + kItemRing);

  constexpr int kProd = kGather ? 4 : 2;  // producer warps (TMA: one for K boxes, one for V boxes)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PATTN_CTA_BEGIN(k2w);
  pdl_wait();  // K5's metadata (or, serial, the previous kernel's work) is complete and visible
  if (p.partition) {
    // two-stream SM partition (as K2): K5's P SMs belong to the prefill kernel while it still
    // has Q blocks to claim; a decode CTA placed there first leaves.  CTA 0 always works.
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
    for (int s = 0; s < nent; ++s) {
      mbar_init(&full[s], kGather ? kProd * 32 : 1);  // gather: one noinc arrive per producer thread
      mbar_init(&empty[s], HB * HGW);
    }
    for (int i = 0; i < kItemRing; ++i) {
      mbar_init(&item_full[i], 1);
      mbar_init(&item_empty[i], HB * HGW + kProd - 1);  // consumers + the other producer warps
    }
    fence_barrier_init();
  }
  __syncthreads();

  const int ngroups = p.Hkv / HB;
  const int n_items = p.hdr[kHdrTotalChunks] * ngroups;
  const int n16 = p.bs / kSub;

  if (kGather && warp < kProd) {
    // ------------------------------------------------------------ gather producers
    // Thread i of the 128 owns key row t = i / 8 of every sub-block and 16-byte chunk ch = i % 8
    // of each 128-byte row segment: per entry it issues HB x D/64 cp.async into the entry's
    // swizzled [head][half][slot][64 d] layout (the TMA box layout) and one noinc arrive.
    const int tid = threadIdx.x, t = tid >> 3, ch = tid & 7;
    const uint64_t policy = l2_policy_evict_first();
    const int esz = (int)sizeof(typename E::T);
    uint32_t s = 0, ph = 0;
    for (uint32_t ni = 0;; ++ni) {
      int it = 0;
      const uint32_t slot = ni % kItemRing;
      if (warp == 0) {
        if (lane == 0) {
          mbar_wait(&item_empty[slot], ((ni / kItemRing) & 1u) ^ 1u);
          it = atomicAdd(p.hdr + kHdrDecodeCounter, 1);
          item_ring[slot] = it;
          mbar_arrive(&item_full[slot]);
        }
        it = __shfl_sync(0xffffffffu, it, 0);
      } else {
        mbar_wait(&item_full[slot], (ni / kItemRing) & 1u);
        it = item_ring[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&item_empty[slot]);
      }
      if (it >= n_items) {
        if (warp == 0 && lane == 0) {
          pdl_trigger();
          atomicExch(p.hdr + kHdrDecodeClaimed, 1);  // (K1's late CTAs may take decode SMs now)
        }
        break;
      }
      const WItem x = wide_item(p, it, ngroups);
      const int32_t* bt = p.block_table + (int64_t)x.b * p.bt_stride;
      const int nsb = (x.k1 - x.k0 + kSub - 1) / kSub;
      for (int j = 0; j < nsb; ++j) {
        // rows past the segment's keys are left unwritten: their scores are masked by select and
        // the consumers zero those V rows
        const int key = x.k0 + j * kSub + t;
        const bool has_row = key < x.k1;
        int64_t row = 0;  // byte offset of (page, slot, first head of the box, chunk)
        if (has_row) {
          const int pg = key / p.bs;
          row = ((int64_t)__ldg(bt + pg) * p.kv_st_blk + (int64_t)(key - pg * p.bs) * p.kv_st_tok +
                 (int64_t)(x.hb * HB) * p.kv_st_head + ch * 8) * esz;
        }
#pragma unroll
        for (int op = 0; op < 2; ++op) {  // K, then V
          mbar_wait(&empty[s], ph ^ 1u);
          if (has_row) {
            const uint8_t* src = static_cast<const uint8_t*>(op ? p.v : p.k) + row;
            const uint32_t dst = smem_u32(ring + (size_t)s * S::kOpBytes) + t * 128 + ((ch ^ (t & 7)) << 4);
#pragma unroll
            for (int h = 0; h < HB; ++h)
#pragma unroll
              for (int hf = 0; hf < S::kHalves; ++hf)
                cp_async_16_hint(dst + h * S::kHeadBytes + hf * S::kHalfBytes,
                                 src + ((int64_t)h * p.kv_st_head + hf * 64) * esz, policy);
          }
          cp_async_mbar_arrive_noinc(&full[s]);
          if (++s == (uint32_t)nent) s = 0, ph ^= 1u;
        }
      }
    }
    return;
  }
  if (!kGather && warp < kProd) {
    // ------------------------------------------------------------ producers
    // warp 0 issues the K boxes (even ring positions), warp 1 the V boxes (odd positions): two
    // issuing threads halve the queueing of the per-request TMA issue cost.  Warp 0 claims the
    // items; warp 1 reads them from the item ring like the consumers.
    const int op = warp;  // 0: K, 1: V
    const CUtensorMap* tm = op ? &tmV : &tmK;
    if (lane == 0) tma_prefetch_desc(tm);
    const uint64_t policy = l2_policy_evict_first();  // K/V are streamed exactly once
    // ring position of this producer's next entry, kept incrementally (nent is a runtime value:
    // g % nent and g / nent would cost an integer division per entry); K(j) at position 2g, V(j)
    // at 2g + 1 of the CTA's sub-block sequence
    uint32_t s = (uint32_t)op % (uint32_t)nent, ph = 0;
    for (uint32_t ni = 0;; ++ni) {
      int it = 0;
      const uint32_t slot = ni % kItemRing;
      if (op == 0) {
        if (lane == 0) {
          mbar_wait(&item_empty[slot], ((ni / kItemRing) & 1u) ^ 1u);
          it = atomicAdd(p.hdr + kHdrDecodeCounter, 1);
          item_ring[slot] = it;
          mbar_arrive(&item_full[slot]);
        }
        it = __shfl_sync(0xffffffffu, it, 0);
      } else {
        mbar_wait(&item_full[slot], (ni / kItemRing) & 1u);
        it = item_ring[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&item_empty[slot]);
      }
      if (it >= n_items) {
        if (op == 0 && lane == 0) {
          pdl_trigger();                              // no more items here: K3 may be scheduled
          atomicExch(p.hdr + kHdrDecodeClaimed, 1);  // and K1's late CTAs may take decode SMs
        }
        break;
      }
      const WItem x = wide_item(p, it, ngroups);
      const int32_t* bt = p.block_table + (int64_t)x.b * p.bt_stride;
      for (int j0 = x.sb0; j0 < x.sb1; j0 += 32) {
        const int n = min(32, x.sb1 - j0);
        const int id = lane < n ? __ldg(bt + (j0 + lane) / n16) : 0;  // 32 sub-blocks' blocks at once
        for (int jj = 0; jj < n; ++jj) {
          const int blk = __shfl_sync(0xffffffffu, id, jj);
          if (lane == 0) {
            const int slot0 = ((j0 + jj) % n16) * kSub;
            mbar_wait(&empty[s], ph ^ 1u);
            mbar_arrive_expect_tx(&full[s], S::kOpBytes);
            tma_load_5d_hint(ring + (size_t)s * S::kOpBytes, tm, &full[s], 0, slot0, 0, x.hb * HB, blk, policy);
          }
          s += 2;  // this producer's next position (positions alternate K, V)
          if (s >= (uint32_t)nent) s -= (uint32_t)nent, ph ^= 1u;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers (one KV head each)
  const int w = (warp - kProd) / HGW, hg = (warp - kProd) % HGW;  // KV head (in the box), head group
  const int r = lane >> 2, c = lane & 3;       // mma fragment coordinates
  const int mat = lane >> 3, mrow = lane & 7;  // ldmatrix source coordinates
  using ET = typename E::T;
  ET* O = static_cast<ET*>(p.out);
  const ET* Q = static_cast<const ET*>(p.q);
  const uint32_t ring_u32 = smem_u32(ring);
  const int G = p.G;
  uint32_t s = 0, ph = 0;  // ring position of the next stage (incremental, as the producer)
  uint32_t ni = 0;  // items consumed (the trace build records it per CTA)
  for (;; ++ni) {
    const uint32_t slot = ni % kItemRing;
    mbar_wait(&item_full[slot], (ni / kItemRing) & 1u);
    const int it = item_ring[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&item_empty[slot]);
    if (it >= n_items) break;
    const WItem x = wide_item(p, it, ngroups);
    const int kvh = x.hb * HB + w;
    const int head0 = kvh * G + hg * 8;
    const int ge = min(8, G - hg * 8);  // query heads of this warp's group

    // Q^T as the B operand of S^T = K . Q^T: b0 = Q[head r][16kc + 2c .. +1], b1 = +8
    uint32_t bq[S::kKC][2];
    {
      const ET* qrow = Q + (int64_t)x.tok * p.q_st_tok + (int64_t)(head0 + r) * p.q_st_head;
#pragma unroll
      for (int kc = 0; kc < S::kKC; ++kc) {
        bq[kc][0] = r < ge ? __ldg(reinterpret_cast<const uint32_t*>(qrow + kc * 16 + 2 * c)) : 0u;
        bq[kc][1] = r < ge ? __ldg(reinterpret_cast<const uint32_t*>(qrow + kc * 16 + 2 * c + 8)) : 0u;
      }
    }
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float acc[S::kKC][4];
#pragma unroll
    for (int t = 0; t < S::kKC; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;

    const int nsb = (x.k1 - x.k0 + kSub - 1) / kSub;
    for (int j = 0; j < nsb; ++j) {
      mbar_wait(&full[s], ph);  // K(j)
      const uint32_t kst = ring_u32 + s * S::kOpBytes + w * S::kHeadBytes;
      const uint32_t ks = s;
      if (++s == (uint32_t)nent) s = 0, ph ^= 1u;
      const uint32_t vs = s, vph = ph;  // V(j): the next entry
      if (++s == (uint32_t)nent) s = 0, ph ^= 1u;
      const uint32_t vst = ring_u32 + vs * S::kOpBytes + w * S::kHeadBytes;
      // two independent accumulation chains (even / odd k-chunks), summed: half the
      // dependent mma latency of one chain (HMMA issues at most every 8 clk per warp)
      float sc[4] = {0.f, 0.f, 0.f, 0.f}, sd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kc = 0; kc < S::kKC; ++kc) {
        const int key = (mat & 1) * 8 + mrow;
        const int dd = kc * 16 + (mat >> 1) * 8;
        const uint32_t addr = kst + (dd >> 6) * S::kHalfBytes + key * 128 + ((((dd & 63) >> 3) ^ (key & 7)) << 4);
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4(addr, a0, a1, a2, a3);
        if (kc & 1)
          E::mma(sd, a0, a1, a2, a3, bq[kc][0], bq[kc][1]);
        else
          E::mma(sc, a0, a1, a2, a3, bq[kc][0], bq[kc][1]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) sc[i] += sd[i];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[ks]);  // K(j) consumed (the ldmatrix results fed the mma)
      mbar_wait(&full[vs], vph);
      const int valid = x.k1 - (x.k0 + j * kSub);  // rows [0, valid) hold this segment's keys
      if (valid < kSub) {
        // zero this head's V rows past the sequence end (NaN * 0 = NaN inside the mma)
        uint8_t* vgen = ring + (size_t)vs * S::kOpBytes + w * S::kHeadBytes;
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
      // Lazy running max (as K1): the exponentials use the running max m unless a score
      // exceeds it by more than 2^8 (log2 domain) -- then, and on an item's first stage
      // (m = -inf), the max is reduced over the 16 keys and O and l are rescaled.  Exact
      // softmax either way (the reference point cancels in acc / l); p <= 2^8 otherwise.  This
      // takes the cross-lane max, two exponentials and the accumulator rescale off the common
      // per-stage path (the consumers are latency-bound: one stage per warp per ~1000 clk).
      float mt0 = fmaxf(s0, s2), mt1 = fmaxf(s1, s3);
      if (__any_sync(0xffffffffu, mt0 > m0 + kLazyMax || mt1 > m1 + kLazyMax)) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          mt0 = fmaxf(mt0, __shfl_xor_sync(0xffffffffu, mt0, o));
          mt1 = fmaxf(mt1, __shfl_xor_sync(0xffffffffu, mt1, o));
        }
        const float mn0 = fmaxf(m0, mt0), mn1 = fmaxf(m1, mt1);  // finite: every sub-block has a valid key
        const float al0 = fast_exp2(m0 - mn0), al1 = fast_exp2(m1 - mn1);
        l0 *= al0;
        l1 *= al1;
        m0 = mn0;
        m1 = mn1;
#pragma unroll
        for (int t = 0; t < S::kKC; ++t) {
          acc[t][0] *= al0;
          acc[t][1] *= al1;
          acc[t][2] *= al0;
          acc[t][3] *= al1;
        }
      }
      const float p0 = fast_exp2(s0 - m0), p1 = fast_exp2(s1 - m1);
      const float p2 = fast_exp2(s2 - m0), p3 = fast_exp2(s3 - m1);
      l0 += p0 + p2;
      l1 += p1 + p3;
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
      if (lane == 0) mbar_arrive(&empty[vs]);
    }

    // ---- this head's result: row sums over the 8 key rows, then output or partial
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, o);
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    const bool h0ok = 2 * c < ge, h1ok = 2 * c + 1 < ge;
    if (x.nseg == 1) {
      const float i0 = 1.f / l0, i1 = 1.f / l1;
      ET* o0 = O + (int64_t)x.tok * p.o_st_tok + (int64_t)(head0 + 2 * c) * p.o_st_head;
      ET* o1 = o0 + p.o_st_head;
#pragma unroll
      for (int t = 0; t < S::kKC; ++t) {
        if (h0ok) {
          o0[16 * t + r] = from_f32<ET>(acc[t][0] * i0);
          o0[16 * t + r + 8] = from_f32<ET>(acc[t][2] * i0);
        }
        if (h1ok) {
          o1[16 * t + r] = from_f32<ET>(acc[t][1] * i1);
          o1[16 * t + r + 8] = from_f32<ET>(acc[t][3] * i1);
        }
      }
    } else {
      const int64_t row0 = (int64_t)x.c * p.Hq + head0 + 2 * c;
      float* a0p = p.part_acc + row0 * D;
      float* a1p = a0p + D;
#pragma unroll
      for (int t = 0; t < S::kKC; ++t) {
        if (h0ok) {
          a0p[16 * t + r] = acc[t][0];
          a0p[16 * t + r + 8] = acc[t][2];
        }
        if (h1ok) {
          a1p[16 * t + r] = acc[t][1];
          a1p[16 * t + r + 8] = acc[t][3];
        }
      }
      if (r == 0) {
        if (h0ok) {
          p.part_m[row0] = m0;
          p.part_l[row0] = l0;
        }
        if (h1ok) {
          p.part_m[row0 + 1] = m1;
          p.part_l[row0 + 1] = l1;
        }
      }
    }
  }
  if (warp == kProd && lane == 0) PATTN_CTA_END(k2w, ni);
}

template <int D, int HB, typename E, bool G, int HGW>
cudaError_t launch_wg(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK, const CUtensorMap& tmV,
                      cudaStream_t stream) {
  auto kern = k2w_decode<D, HB, E, G, HGW>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), dl.smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3(dl.grid), dim3((HB * HGW + (G ? 4 : 2)) * 32), dl.smem, stream, tmK, tmV, p,
                    dl.stages);
}
template <int D, int HB, typename E>
cudaError_t launch_w(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK, const CUtensorMap& tmV,
                     cudaStream_t stream) {
  if (p.G > 8)
    return p.decode_gather ? launch_wg<D, HB, E, true, 2>(p, dl, tmK, tmV, stream)
                           : launch_wg<D, HB, E, false, 2>(p, dl, tmK, tmV, stream);
  return p.decode_gather ? launch_wg<D, HB, E, true, 1>(p, dl, tmK, tmV, stream)
                         : launch_wg<D, HB, E, false, 1>(p, dl, tmK, tmV, stream);
}

template <int D, typename E>
cudaError_t launch_wd(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK, const CUtensorMap& tmV,
                      cudaStream_t stream) {
  switch (p.decode_hb) {
    case 8: return launch_w<D, 8, E>(p, dl, tmK, tmV, stream);
    case 4: return launch_w<D, 4, E>(p, dl, tmK, tmV, stream);
    case 2: return launch_w<D, 2, E>(p, dl, tmK, tmV, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int wide_decode_heads(int Hkv, int G) {
  if (G > 16) return 0;  // G <= 16: one or two head groups of <= 8 query heads per KV head
  const char* e = getenv("PATTN_DECODE_WIDE_HB");  // sweeps: cap on heads per box
  int cap = (e && *e) ? atoi(e) : 8;
  for (int hb = 8; hb >= 2; hb >>= 1)
    if (hb <= cap && Hkv % hb == 0) return hb;
  return 0;
}

// One CTA per SM (the ring takes most of shared memory): ~192 KB of stages, a multiple of the
// 2 x 16 x HB x D x 2 B stage.
DecodeLaunch plan_decode_wide(const Params& p, int num_sms, size_t max_smem) {
  DecodeLaunch dl;
  dl.consumer_warps = p.decode_hb * (p.G > 8 ? 2 : 1);
  const size_t entry = (size_t)kSub * p.decode_hb * p.D * 2;  // one operand box
  const size_t fixed = 1024 /*align slack*/ + 2 * kItemRing * sizeof(uint64_t) + kItemRing * sizeof(int) + 64;
  const size_t cap = (max_smem < 227 * 1024 ? max_smem : 227 * 1024);
  const char* e = getenv("PATTN_DECODE_RING_KB");
  size_t want = (size_t)((e && *e) ? atoi(e) : 224) * 1024;
  if (want + fixed > cap) want = cap - fixed;
  int st = (int)(want / (entry + 16));
  if (st > 32) st = 32;
  if (st < 4) st = 4;
  dl.stages = st;  // ring entries (operand boxes)
  dl.smem = fixed + (size_t)st * (entry + 16);
  const long long max_items = (long long)p.max_chunks * (p.Hkv / p.decode_hb);
  const char* es = getenv("PATTN_DECODE_SMS");
  const long long g = (long long)std::min(num_sms, std::max(1, (es && *es) ? atoi(es) : num_sms));
  dl.grid = (int)(max_items < g ? max_items : g);
  if (dl.grid < 1) dl.grid = 1;
  return dl;
}

cudaError_t launch_decode_wide(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK,
                               const CUtensorMap& tmV, cudaStream_t stream) {
  if (p.D == 128) return p.dtype == 2 ? launch_wd<128, EltF16>(p, dl, tmK, tmV, stream)
                                      : launch_wd<128, EltBf16>(p, dl, tmK, tmV, stream);
  if (p.D == 64) return p.dtype == 2 ? launch_wd<64, EltF16>(p, dl, tmK, tmV, stream)
                                     : launch_wd<64, EltBf16>(p, dl, tmK, tmV, stream);
  return cudaErrorInvalidValue;
}

}  // namespace pattn
