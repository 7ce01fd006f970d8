// K1 -- prefill / long-Q Q-block kernel on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// PAPER.md §4.4 "Prefill and GQA Optimization" (App. B): a Q block packs
// BLOCK_Q consecutive query tokens x the G query heads that share one KV head into a
// BLOCK_M-row tile (token-major / head-minor, reading R8), so every K/V tile is loaded once
// per Q block and shared by all rows.  Here BLOCK_M = 256 = two 128-row halves (a, b), each
// its own UMMA M=128 accumulator, so BLOCK_Q = 2 * floor(128/G) (padding rows when G does not
// divide 128).  KV tiles of 64 keys = 4 sub-blocks of 16 keys gathered through the block
// table -- one TMA box per sub-block from any block size that is a multiple of 16, or, for
// other block sizes, row by row with cp.async (kGather) -- tile size decoupled from
// BLOCK_SIZE (§4.6).  The tiled (online) softmax of §4.1 runs between
// the two contractions.
//
// One CTA per SM, persistent over (Q block, KV head) work items (static launch grid,
// P:401-406), longest (last) Q blocks first, claimed dynamically from a global counter (reset
// by K5) by a scheduler warp that publishes them to the other roles through a shared-memory
// ring, so a CTA that shares the GPU with the decode kernel (two streams) or drew short items
// simply claims fewer.  Warp roles (16 warps, setmaxnreg-rebalanced registers):
//   warps 0, 2 / 3, 12  TMA producers of the K / V rings (two sub-blocks each per tile;
//                sub-blocks past the visible range are requested out of bounds: zero fill)
//   warp 14      Q producer (both halves), warp 13 item scheduler, warp 2 also allocates TMEM
//   warps 1, 15  MMA issuers for half a / b (one elected lane): S_h(j) = Q_h K^T into S buffer
//                j & 1 (SS mode), then PV_h(j-1): O_h += P_h V with P (bf16) in TMEM aliased on
//                its S buffer (TS mode) -- the softmax of tile j overlaps PV(j-1).
//   TMEM (512 columns): S_a0 | S_a1 | S_b0 | S_b1 (64 each) | O_a | O_b (128 each, D = 128)
//   warps 4..7 / 8..11  softmax warpgroups of half a / b (thread r owns row r = TMEM lane r):
//                tcgen05.ld of the S row, causal mask on diagonal / tail tiles (row limit
//                ctx+i+1), max, exp2, row sum; lazy rescale of O in TMEM only when
//                the running max grows by > 2^8 (exact: p <= 256 otherwise); P written back into
//                TMEM with tcgen05.st; epilogue O / l -> bf16 -> 128B-swizzled staging -> TMA store.
// V rows past the sequence end inside the last sub-block may hold NaN (reading R13): the
// softmax warpgroups zero them in shared memory before releasing P.
#include "common.cuh"
#include "kernels.h"

#include "trace.cuh"
PATTN_CTA_TRACE_DEFINE(k1)
#ifdef PATTN_TRACE
// debug timeline of CTA 0: one array per recording thread (no atomics: fire-and-forget stores)
// slot = (role, index): role 0 MMA thread, 1/2 softmax WG a/b thread 0, 3/4 K/V producer lane 0
__device__ unsigned long long g_k1_trace[5][2 * 2048];
__device__ unsigned int g_k1_trace_n[5];
#define PATTN_K1_TRACE_ROLE(role, cnt, code)                          \
  do {                                                                \
    if (blockIdx.x == 0 && (role) >= 0 && (cnt) < 2048) {             \
      g_k1_trace[role][2 * (cnt)] = clock64();                        \
      g_k1_trace[role][2 * (cnt) + 1] = (code);                       \
      g_k1_trace_n[role] = ++(cnt);                                   \
    }                                                                 \
  } while (0)
extern "C" __attribute__((visibility("default"))) int pattn_debug_k1_trace(unsigned long long* host, int cap, int reset) {
  unsigned int n[5];
  cudaMemcpyFromSymbol(n, g_k1_trace_n, sizeof(n));
  static unsigned long long tmp[5][2 * 2048];
  cudaMemcpyFromSymbol(tmp, g_k1_trace, sizeof(tmp));
  int k = 0;
  for (int r = 0; r < 5; ++r)
    for (unsigned i = 0; i < n[r] && i < 2048 && k < cap; ++i, ++k) {
      host[2 * k] = tmp[r][2 * i];
      host[2 * k + 1] = tmp[r][2 * i + 1];
    }
  if (reset) {
    unsigned int z[5] = {0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_k1_trace_n, z, sizeof(z));
  }
  return k;
}
#define PATTN_K1_TRACE(code) PATTN_K1_TRACE_ROLE(trace_role, trace_cnt, code)
#else
#define PATTN_K1_TRACE(code) \
  do {                       \
  } while (0)
#endif

namespace pattn {
namespace {

constexpr int kHalfM = 128;    // rows per half (one UMMA M)
constexpr int kM = 2 * kHalfM; // BLOCK_M
constexpr int kN = 64;         // keys per KV tile
constexpr int kThreads = 512;  // 16 warps
// setmaxnreg budgets (16-warp layout): warpgroup 0 (producers, MMA a), warpgroups 1-2
// (softmax), warpgroup 3 (V producer, scheduler, Q producer, MMA b); 128 (a + d) + 256 s = 65536
#ifndef PATTN_K1_REG_WG0
#define PATTN_K1_REG_WG0 56
#endif
#ifndef PATTN_K1_REG_SOFTMAX
#define PATTN_K1_REG_SOFTMAX 208
#endif
#ifndef PATTN_K1_REG_WG3
#define PATTN_K1_REG_WG3 40
#endif
constexpr int kRegWG0 = PATTN_K1_REG_WG0, kRegSoftmax = PATTN_K1_REG_SOFTMAX, kRegWG3 = PATTN_K1_REG_WG3;
// setmaxnreg only redistributes the CTA's launch allocation
static_assert(128 * (kRegWG0 + kRegWG3) + 256 * kRegSoftmax <= 65536, "register budget");
// K / V tile layout: sub-block i (16 keys) = [8-slot group g][d half h][8 slots][64 d], i.e.
// 8-key group G = 2i+g at G*kGroup + h*1024 (SW128 atoms of 8 rows x 128 B); kGroup = 16*D B.
#ifndef PATTN_K1_KST
#define PATTN_K1_KST 3
#endif
#ifndef PATTN_K1_VST
#define PATTN_K1_VST 3
#endif
constexpr int kKStages = PATTN_K1_KST;
constexpr int kVStages = PATTN_K1_VST;  // V waits on PV (later than S), so it gets the deeper ring
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale O only if the max grows by > 2^8
constexpr uint32_t kBarBlock = 512;        // barriers + the item ring

// Head-dim dependent sizes and the shared-memory map (offsets from a 1024-aligned base).
template <int D>
struct K1Shape {
  static_assert(D == 64 || D == 128, "head_dim");
  static constexpr int kHalves = D / 64;                   // 64-wide (128-byte) d halves
  static constexpr uint32_t kQTile = kHalfM * D * 2;       // one 128-row half of the Q block (32 / 16 KB)
  static constexpr uint32_t kHalf = kHalfM * 64 * 2;       // 16 KB: one 64-wide d half of a Q half
  static constexpr uint32_t kTile = kN * D * 2;            // one K or V tile (64 keys: 16 / 8 KB)
  static constexpr uint32_t kSub16Bytes = 16 * D * 2;      // one 16-key sub-block (4 / 2 KB)
  static constexpr uint32_t kGroup = 8 * D * 2;            // one 8-key group (2 / 1 KB)
  static constexpr uint32_t kOffQ = 0;                     // half a, then half b
  static constexpr uint32_t kOffK = kOffQ + 2 * kQTile;
  static constexpr uint32_t kOffV = kOffK + kKStages * kTile;
  // epilogue staging, 128B-swizzled as the out TMA map expects: per warp 32 rows x 128 B per
  // 64-wide d half, all halves staged at once (no read wait in between)
  static constexpr uint32_t kStageWarp = 4096 * kHalves;
  static constexpr uint32_t kStageHalf = 4 * kStageWarp;
  static constexpr uint32_t kOffStage = kOffV + kVStages * kTile;
  static constexpr uint32_t kOffBar = kOffStage + 2 * kStageHalf;
  static constexpr uint32_t kSmemBytes = kOffBar + kBarBlock + 1024;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

// TMEM columns
constexpr uint32_t kTmemS = 0;    // S buffer (half x, tile parity y) at x*128 + y*64 (P aliased on its first 32 cols)
constexpr uint32_t kTmemO = 256;  // O_x at 256 + x*128

// Item ring depth: the scheduler runs kItemRing - 1 items ahead.  Claiming an item costs a
// global atomic plus dependent metadata / block-table loads (~3-4k clk), more than a short
// (1-2 tile) item lasts, so a 2-deep ring exposed it at the tail of the queue.
#ifndef PATTN_K1_ITEM_RING
#define PATTN_K1_ITEM_RING 2  // measured: 4 -> -5%, 8 -> -10% (claiming ahead unbalances the tail)
#endif
constexpr int kItemRing = PATTN_K1_ITEM_RING;

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2][2], p_full[2], pv_done[2], o_empty[2];
  // dynamic work queue (see ItemSlot)
  uint64_t item_full[kItemRing], item_empty[kItemRing];
  uint32_t tmem_base;
};

// One MMA-issuing warp per half (warp 1: half a, warp 15: half b) so that one half's chain
// S(j) -> softmax(j) -> PV(j) never waits behind the other half's softmax.
constexpr int kMmaWarps = 2;
constexpr int kItemConsumers = 15;  // warps 0-3, 12, 14, 15 and the 8 softmax warps

struct Item {
  int b, kvh, q0, qlen, L, ctx, tok0, ntok, kv_end, ntiles;
};
// Scheduler warp 13 claims the next item from the global counter (longest first), decodes it
// and fetches the block-table entries of its first KV tile while the CTA still works on the
// current item, so that neither the claim's atomic nor the dependent metadata / block-table
// loads sit on the critical path at item boundaries.  ntiles < 0 ends the stream.
struct ItemSlot {
  Item x;
  int ids[8];  // paged block of each 16-key sub-block of KV tile 0 (num_blocks: past the end)
};
constexpr uint32_t kOffItems = sizeof(Bars);
static_assert(sizeof(Bars) + kItemRing * sizeof(ItemSlot) <= kBarBlock, "barrier block");

__device__ __forceinline__ Item prefill_item(const Params& p, int total_qb, int qb_uniform, int qb_group, int it,
                                             int lane) {
  Item x;
  // Claim order, longest key range first: the Q blocks of a sequence from its last one; when all
  // Q-block sequences have the same number u of Q blocks (K5), rank by rank across a group of
  // g sequences (the last Q block of each, then each second-to-last, ...; groups in order, g
  // from an L2 budget) -- the per-sequence order alone leaves a late sequence's longest items
  // for the end of the queue (config 3 measured a 57 us spread of K1's CTA end times).
  const int q = it / p.Hkv;
  int j = total_qb - 1 - q;
  if (qb_uniform > 0) {
    const int u = qb_uniform, m = total_qb / u, gu = qb_group * u;
    const int gi = q / gu, qq = q - gi * gu, gs = min(qb_group, m - gi * qb_group);
    const int r = qq / gs, i = qq - r * gs;
    j = (gi * qb_group + i) * u + (u - 1 - r);
  }
  x.kvh = it % p.Hkv;
  x.b = upper_bound_minus1_warp(p.cu_qb, p.B, j, lane);  // App. B P:46 (warp-cooperative search)
  const int qblk = j - __ldg(p.cu_qb + x.b);
  x.q0 = __ldg(p.cu_seqlens_q + x.b);
  x.qlen = __ldg(p.cu_seqlens_q + x.b + 1) - x.q0;
  x.L = __ldg(p.seq_lens + x.b);
  x.ctx = x.L - x.qlen;
  x.tok0 = qblk * p.block_q;
  x.ntok = min(p.block_q, x.qlen - x.tok0);
  x.kv_end = x.ctx + x.tok0 + x.ntok;  // keys visible to the Q block's last row
  x.ntiles = (x.kv_end + kN - 1) / kN;
  return x;
}

// O[tmem] (+)= A[tmem] * B[smem desc]; kind::f16, A (P) K-major in TMEM.
PATTN_DEVICE void tc_mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}

// Consumer side of the item ring (whole warp): the n-th item of this CTA (and, for the
// producers, the block ids of its first tile).
PATTN_DEVICE Item next_item(Bars& bar, const ItemSlot* ring, uint32_t n, int lane, int* ids0 = nullptr) {
  const uint32_t slot = n % kItemRing;
  mbar_wait(&bar.item_full[slot], (n / kItemRing) & 1u);
  const volatile ItemSlot* e = ring + slot;
  Item x;
  x.b = e->x.b;
  x.kvh = e->x.kvh;
  x.q0 = e->x.q0;
  x.qlen = e->x.qlen;
  x.L = e->x.L;
  x.ctx = e->x.ctx;
  x.tok0 = e->x.tok0;
  x.ntok = e->x.ntok;
  x.kv_end = e->x.kv_end;
  x.ntiles = e->x.ntiles;
  if (ids0) *ids0 = e->ids[lane & 7];
  __syncwarp();
  if (lane == 0) mbar_arrive(&bar.item_empty[slot]);
  return x;
}

// kGather: block sizes that are not a multiple of 16 (no 16-key TMA box fits a page): the four
// producer warps gather each K / V tile row by row with 16-byte cp.async into the same swizzled
// layout (one block-table lookup per key row; keys past the Q block's visible range zero-filled),
// completing on the stage's mbarrier with cp.async.mbarrier.arrive.noinc (64 producer threads per
// operand); everything else is unchanged.
template <int D, typename E, bool kGather>
__global__ void __launch_bounds__(kThreads, 1)
    k1_prefill(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO,
               const __grid_constant__ KvHeadMaps maps, Params p) {
  using Sh = K1Shape<D>;
  constexpr uint32_t kOffQ = Sh::kOffQ, kOffK = Sh::kOffK, kOffV = Sh::kOffV, kOffStage = Sh::kOffStage,
                     kOffBar = Sh::kOffBar, kQTile = Sh::kQTile, kHalf = Sh::kHalf, kTile = Sh::kTile,
                     kSub16Bytes = Sh::kSub16Bytes, kStageWarp = Sh::kStageWarp, kGroup = Sh::kGroup;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars& bar = *reinterpret_cast<Bars*>(smem + kOffBar);
  ItemSlot* ring = reinterpret_cast<ItemSlot*>(smem + kOffBar + kOffItems);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PATTN_CTA_BEGIN(k1);
  pdl_wait();  // K5's metadata (and the SM partition) is complete and visible
  // two-stream SM partition (K5's choice): K1 works on the P lowest SM IDs; a CTA placed on
  // another SM leaves it to the decode kernel at once.  Keyed on the physical SM (not blockIdx:
  // the round-1 rule, launch-order dependent), so it holds whichever kernel the hardware (or a
  // replayed CUDA graph, whose two branches start in either order) launches first.  CTA 0
  // always works (progress guarantee).  A CTA that reaches a decode SM only after the decode kernel's queue is empty (a replayed graph
  // may start the decode branch first: K1's CTAs for those SMs then wait behind the decode CTAs)
  // stays and takes prefill items -- K1 then spreads onto the SMs the decode side has finished.
  if (p.partition && blockIdx.x != 0 && !partition_prefill_sm(sm_id(), p.hdr[kHdrPrefillCtas], p.num_sms) &&
      *reinterpret_cast<volatile int*>(p.hdr + kHdrDecodeClaimed) == 0)
    return;
#ifdef PATTN_TRACE
  const int trace_role = warp == 15 ? -1 : warp == 1 ? 0 : warp == 0 ? 3 : warp == 3 ? 4 : warp == 4 ? 1 : 2;
  unsigned int trace_cnt = 0;
#endif

  if (threadIdx.x == 0) {
    mbar_init(&bar.q_full, 1);
    mbar_init(&bar.q_empty, kMmaWarps);
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&bar.k_full[s], kGather ? 64 : 1);
      mbar_init(&bar.k_empty[s], kMmaWarps);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&bar.v_full[s], kGather ? 64 : 1);
      mbar_init(&bar.v_empty[s], kMmaWarps);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&bar.s_full[h][0], 1);
      mbar_init(&bar.s_full[h][1], 1);
      mbar_init(&bar.p_full[h], kHalfM);
      mbar_init(&bar.pv_done[h], 1);
      mbar_init(&bar.o_empty[h], kHalfM);
    }
    for (int i = 0; i < kItemRing; ++i) {
      mbar_init(&bar.item_full[i], 1);
      mbar_init(&bar.item_empty[i], kItemConsumers);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(&bar.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;

  const int total_qb = p.hdr[kHdrTotalQBlocks];
  const int qb_uniform = p.hdr[kHdrQbUniform], qb_group = p.hdr[kHdrQbGroup];
  const int n_items = total_qb * p.Hkv;
  const int G = p.G;
  const int bq_half = p.block_q / 2;  // tokens per 128-row half

  // register rebalancing per warpgroup: warpgroup 0 (producers, MMA) 56, softmax warpgroups
  // 1-2 208, warpgroup 3 (producer + spares) 40: 128*56 + 256*208 + 128*40 = 65536

  if (warp == 0 || warp == 2 || warp == 3 || warp == 12) {
    // ================================================================ TMA producers
    // warp 0: Q and sub-blocks 0-3 of every K tile, warp 2: K sub-blocks 4-7, warp 3: V
    // sub-blocks 0-3, warp 12: V sub-blocks 4-7.  K and V rings are independent (a V stage
    // still in use by PV never delays the next K tile the S MMA waits for) and the per-box
    // TMA issue cost (~150 clk) is spread over four warps.
    if (warp < 4)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegWG0) : "memory");
    else
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegWG3) : "memory");
    const int kv = (warp == 3 || warp == 12) ? 1 : 0;
    const bool owner = warp == 0 || warp == 3;  // arms the stage barrier with the tile's byte count
    const int i_lo = owner ? 0 : kN / 32, i_hi = i_lo + kN / 32;  // 2 sub-blocks per warp
    // A 128-key tile = 8 sub-blocks of 16 keys; sub-block idx is slots [(idx % n16)*16, +16)
    // of paged block bt[idx / n16] (any block size that is a multiple of 16).  One 4 KB TMA
    // box per sub-block (per-head 5-D map); the warp's 4 boxes are issued by lanes 0-3
    // together.
    constexpr int nbt = kN / 16;
    const int n16 = p.bs / 16;
    const uint64_t pol_kv = l2_policy_evict_last();  // K/V tiles are re-read by the sequence's other Q blocks
    const int nst = kv ? kVStages : kKStages;
    uint32_t ic = 0, cnt = 0;
    if constexpr (kGather) {
      static_assert(kN == 64, "one key row per producer thread");
      const int t = (owner ? 0 : 32) + lane;  // this thread's key row of every tile
      constexpr int esz = (int)sizeof(typename E::T);
      for (;; ++ic) {
        const Item x = next_item(bar, ring, ic, lane);
        if (x.ntiles < 0) break;
        const uint8_t* gbase = static_cast<const uint8_t*>(kv ? p.v : p.k) + (int64_t)x.kvh * p.kv_st_head * esz;
        const int32_t* bt = p.block_table + (int64_t)x.b * p.bt_stride;
        // the block-table entry of this thread's row, one tile ahead (its load latency overlaps
        // the current tile's copies)
        int id_next = t < x.kv_end ? __ldg(bt + t / p.bs) : 0;
        for (int jt = 0; jt < x.ntiles; ++jt) {
          const uint32_t s = cnt % nst, ph = (cnt / nst) & 1u;
          uint64_t* fullb = kv ? &bar.v_full[s] : &bar.k_full[s];
          uint64_t* emptyb = kv ? &bar.v_empty[s] : &bar.k_empty[s];
          const uint32_t dst = smem_u32(smem + (kv ? kOffV : kOffK) + s * kTile) + (t >> 3) * kGroup + (t & 7) * 128;
          const int key = jt * kN + t;
          const int id = id_next;
          id_next = (jt + 1 < x.ntiles && key + kN < x.kv_end) ? __ldg(bt + (key + kN) / p.bs) : 0;
          const uint8_t* src = gbase;
          int bytes = 0;  // 0: zero-fill (keys past the visible range, and past the sequence end)
          if (key < x.kv_end) {
            src = gbase + ((int64_t)id * p.kv_st_blk + (int64_t)(key % p.bs) * p.kv_st_tok) * esz;
            bytes = 16;
          }
          if (lane == 0) mbar_wait(emptyb, ph ^ 1u);
          __syncwarp();
#pragma unroll
          for (int c = 0; c < D / 8; ++c)  // 16-byte chunk c of the row: d half c / 8, chunk c % 8 (swizzled)
            cp_async_16_zfill_hint(dst + (c >> 3) * 1024 + (((c & 7) ^ (t & 7)) << 4), src + (bytes ? c * 16 : 0),
                                   bytes, pol_kv);
          cp_async_mbar_arrive_noinc(fullb);
          ++cnt;
        }
      }
    } else
    for (;; ++ic) {
      int id0;
      const Item x = next_item(bar, ring, ic, lane, &id0);
      if (x.ntiles < 0) break;
      const CUtensorMap* tm = kv ? &maps.v[x.kvh] : &maps.k[x.kvh];
      if (lane == 0) tma_prefetch_desc(tm);
      const int32_t* bt = p.block_table + (int64_t)x.b * p.bt_stride;
      const int nsb_valid = (x.kv_end + 15) / 16;  // sub-blocks holding visible keys
      int id_next = id0;  // tile 0: fetched by the scheduler
      for (int jt = 0; jt < x.ntiles; ++jt) {
        const int id_cur = id_next;
        const int sb_next = (jt + 1) * nbt + lane;
        id_next = (jt + 1 < x.ntiles && lane < nbt && sb_next < nsb_valid) ? __ldg(bt + sb_next / n16) : p.num_blocks;
        const uint32_t s = cnt % nst, ph = (cnt / nst) & 1u;
        uint64_t* fullb = kv ? &bar.v_full[s] : &bar.k_full[s];
        uint64_t* emptyb = kv ? &bar.v_empty[s] : &bar.k_empty[s];
        uint8_t* base = smem + (kv ? kOffV : kOffK) + s * kTile;
        const int i = i_lo + (lane & 1);
        const int blk = __shfl_sync(0xffffffffu, id_cur, i);
        if (lane == 0) {
          if (owner) PATTN_K1_TRACE(24 + kv);
          mbar_wait(emptyb, ph ^ 1u);
          if (owner) mbar_arrive_expect_tx(fullb, kTile);
          if (owner) PATTN_K1_TRACE(20 + kv);
        }
        __syncwarp();
        if (lane < kN / 32) {
          const int grp0 = ((jt * nbt + i) % n16) * 2;  // first 8-slot group of the sub-block
          tma_load_5d_hint(base + i * kSub16Bytes, tm, fullb, 0, 0, 0, grp0, blk, pol_kv);
        }
        __syncwarp();
        if (lane == 0 && owner) PATTN_K1_TRACE(22 + kv);
        ++cnt;
      }
    }
  } else if (warp == 1 || warp == 15) {
    // ================================================================ MMA issuer(s)
    // The whole warp runs the schedule (waits, descriptor arithmetic stay warp-uniform, in
    // uniform registers); one elected lane issues each tcgen05.mma / commit.  With two MMA
    // warps, warp 1 issues half a's S and PV and warp 15 half b's; K / V / Q stages are
    // released when both have committed (the empty barriers count kMmaWarps arrivals).
    if (warp == 1)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegWG0) : "memory");
    else
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegWG3) : "memory");  // warpgroup 3
    const int h_lo = warp == 15 ? 1 : 0;
    const int h_hi = h_lo + 1;
    constexpr uint32_t idS = idesc_f16kind_f32(kHalfM, kN, 0, 0, E::kUmmaFmt);   // Q (K-major) x K (K-major)
    constexpr uint32_t idPV = idesc_f16kind_f32(kHalfM, D, 0, 1, E::kUmmaFmt);  // P (TMEM, K-major) x V (MN-major)
    // smem descriptors: start-address field = addr >> 4, so desc(base + off) = desc(base) + (off >> 4)
    const uint64_t dQ = smem_desc_sw128(sbase + kOffQ, 16, 1024);
    const uint64_t dK = smem_desc_sw128(sbase + kOffK, 16, kGroup);     // 8-key groups kGroup apart
    const uint64_t dV = smem_desc_sw128(sbase + kOffV, 1024, kGroup);   // d halves 1 KB apart
    const bool leader = elect_one();
    uint32_t ic = 0, kc = 0, vc = 0;
    uint32_t pcnt = 0u;  // PV iterations issued (the same count for every half this warp serves)
    for (;; ++ic) {
      const Item x = next_item(bar, ring, ic, lane);
      if (x.ntiles < 0) break;
      if (leader) PATTN_K1_TRACE(40);
      mbar_wait(&bar.q_full, ic & 1u);
      if (leader) PATTN_K1_TRACE(41);
      tc_fence_after();
      // Iteration jt: S_a(jt), S_b(jt) into S buffer jt&1 of each half, then PV_a(jt-1),
      // PV_b(jt-1) from buffer (jt-1)&1.  S_h(jt) overwrites P_h(jt-2), whose PV was issued
      // one iteration earlier (tcgen05 ops execute in issue order), so the softmax of tile
      // jt overlaps the PV of tile jt-1 instead of waiting for it.
      for (int jt = 0; jt <= x.ntiles; ++jt) {
        const bool do_s = jt < x.ntiles, do_pv = jt > 0;
        if (do_s) {
          const uint32_t ks = kc % kKStages;
          mbar_wait(&bar.k_full[ks], (kc / kKStages) & 1u);
          if (leader) PATTN_K1_TRACE(1);
          tc_fence_after();
          if (leader) {
            for (int h = h_lo; h < h_hi; ++h) {
              const uint32_t tS = tmem + kTmemS + 128 * h + 64 * (jt & 1);
              const uint64_t dq = dQ + ((h * kQTile) >> 4), dk = dK + ((ks * kTile) >> 4);
#pragma unroll
              for (int k = 0; k < D / 16; ++k) {
                const uint32_t offq = ((k >> 2) * kHalf + (k & 3) * 32) >> 4;
                const uint32_t offk = ((k >> 2) * 1024 + (k & 3) * 32) >> 4;
                tc_mma_f16_ss(tS, dq + offq, dk + offk, idS, k > 0 ? 1u : 0u);
              }
              PATTN_K1_TRACE(7 + h);
              tc_commit(&bar.s_full[h][jt & 1]);
            }
            tc_commit(&bar.k_empty[ks]);
            if (jt == x.ntiles - 1) tc_commit(&bar.q_empty);
          }
          __syncwarp();
          ++kc;
        }
        if (do_pv) {
          const uint32_t vs = vc % kVStages;
          mbar_wait(&bar.v_full[vs], (vc / kVStages) & 1u);
          if (leader) PATTN_K1_TRACE(2);
          for (int h = h_lo; h < h_hi; ++h) {
            const uint32_t tP = tmem + kTmemS + 128 * h + 64 * ((jt - 1) & 1), tO = tmem + kTmemO + 128 * h;
            mbar_wait(&bar.p_full[h], pcnt & 1u);
            if (jt == 1) mbar_wait(&bar.o_empty[h], (ic & 1u) ^ 1u);
            tc_fence_after();
            if (leader) {
              PATTN_K1_TRACE(3 + h);
              const uint64_t dv = dV + ((vs * kTile) >> 4);
#pragma unroll
              for (int k = 0; k < kN / 16; ++k) {
                tc_mma_f16_ts(tO, tP + 8 * k, dv + ((k * kSub16Bytes) >> 4), idPV, (jt > 1 || k > 0) ? 1u : 0u);
              }
              PATTN_K1_TRACE(5 + h);
              tc_commit(&bar.pv_done[h]);
            }
            __syncwarp();
          }
          ++pcnt;
          if (leader) tc_commit(&bar.v_empty[vs]);
          __syncwarp();
          ++vc;
        }
      }
    }
  } else if (warp == 13 || warp == 14) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegWG3) : "memory");  // warpgroup 3 (13, 14)
    if (warp == 13) {
      // ================================================================ item scheduler
      const int n16 = p.bs / 16;
      for (uint32_t n = 0;; ++n) {
        const uint32_t slot = n % kItemRing;
        int it = 0;
        if (lane == 0) {
          mbar_wait(&bar.item_empty[slot], ((n / kItemRing) & 1u) ^ 1u);
          it = atomicAdd(p.hdr + kHdrPrefillCounter, 1);
        }
        it = __shfl_sync(0xffffffffu, it, 0);
        volatile ItemSlot* e = ring + slot;
        if (it < n_items) {
          const Item x = prefill_item(p, total_qb, qb_uniform, qb_group, it, lane);
          const int nsb_valid = (x.kv_end + 15) / 16;
          // (gathered producers look their rows up themselves: no prefetch, and n16 = 0 there)
          const int id = (!kGather && lane < 8 && lane < nsb_valid)
                             ? __ldg(p.block_table + (int64_t)x.b * p.bt_stride + lane / n16)
                             : p.num_blocks;
          int ids[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) ids[q] = __shfl_sync(0xffffffffu, id, q);
          if (lane == 0) {  // one writer: program order before its release (the arrive below)
#pragma unroll
            for (int q = 0; q < 8; ++q) e->ids[q] = ids[q];
            e->x.b = x.b;
            e->x.kvh = x.kvh;
            e->x.q0 = x.q0;
            e->x.qlen = x.qlen;
            e->x.L = x.L;
            e->x.ctx = x.ctx;
            e->x.tok0 = x.tok0;
            e->x.ntok = x.ntok;
            e->x.kv_end = x.kv_end;
            e->x.ntiles = x.ntiles;
          }
        } else if (lane == 0) {
          e->x.ntiles = -1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.item_full[slot]);
        if (it >= n_items) break;
      }
    } else if (warp == 14) {
      // ================================================================ Q producer
      // Its own warp, so that waiting for the single Q buffer to drain (the current item's
      // last S MMA) never holds back the K/V producers' prefetch of the next item's tiles.
      if (lane == 0) tma_prefetch_desc(&tmQ);
      for (uint32_t ic = 0;; ++ic) {
        const Item x = next_item(bar, ring, ic, lane);
        if (x.ntiles < 0) break;
        if (lane == 0) {
          mbar_wait(&bar.q_empty, (ic & 1u) ^ 1u);
          mbar_arrive_expect_tx(&bar.q_full, 2u * Sh::kHalves * (uint32_t)(bq_half * G) * 128u);  // halves x d-halves
          for (int h = 0; h < 2; ++h) {
            const int tok = x.q0 + x.tok0 + h * bq_half;
#pragma unroll
            for (int dh = 0; dh < Sh::kHalves; ++dh)
              tma_load_4d(smem + kOffQ + h * kQTile + dh * kHalf, &tmQ, &bar.q_full, 64 * dh, 0, x.kvh, tok);
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ================================================================ softmax / correction / epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegSoftmax) : "memory");
    const int h = (warp - 4) >> 2;        // half a (0) or b (1)
    const int r = 32 * (warp & 3) + lane;  // row within the half == TMEM lane
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t tS0 = tmem + kTmemS + 128 * h + lane_off;
    const uint32_t tO = tmem + kTmemO + 128 * h + lane_off;
    const bool lead = r == 0;  // trace recorder
    uint32_t tc = 0, vc = 0;  // tiles seen by this warpgroup (== PV count of this half)
    uint32_t sc0 = 0u, sc1 = 0u;  // completed phases observed per S buffer (scalars: a runtime-indexed
                                  // array would live in local memory inside the tile loop)
    using OutT = typename E::T;
    OutT* O = static_cast<OutT*>(p.out);
    const float cs = p.scale_log2;
    const float ca = fmaxf(fabsf(cs), 1e-30f);  // scale 0: -inf * 0 would be NaN; 1e-30 * s ~ 0
    uint32_t ic = 0;
    for (;; ++ic) {
      const Item x = next_item(bar, ring, ic, lane);
      if (x.ntiles < 0) break;
      const int tk = h * bq_half + r / G;  // token of this row within the Q block
      // G not dividing 128: rows r >= bq_half * G of a half are padding (their Q rows are never
      // loaded); they see no key (fully masked, never stored)
      const bool row_live = r < bq_half * G;
      const bool row_valid = row_live && tk < x.ntok;
      const int row_lim = row_live ? min(x.ctx + x.tok0 + tk + 1, x.kv_end) : 0;  // keys [0, row_lim) visible
      const int nsb_valid = (x.kv_end + 15) / 16;                  // 16-key sub-blocks fetched
      float m_run = -INFINITY, l_run = 0.f;
      float s[kN];
      for (int jt = 0; jt < x.ntiles; ++jt) {
        const int sb = jt & 1;  // S buffer of this tile (P is written back over it)
        const uint32_t tS = tS0 + 64 * sb;
        mbar_wait(&bar.s_full[h][sb], (sb ? sc1 : sc0) & 1u);
        sc0 += sb ? 0u : 1u;
        sc1 += sb ? 1u : 0u;
        if (lead) PATTN_K1_TRACE(10 + h);
        tc_fence_after();
        {
          uint32_t* su = reinterpret_cast<uint32_t*>(s);
          PATTN_TMEM_LD32(tS + 0, (su + 0));
          PATTN_TMEM_LD32(tS + 32, (su + 32));
          tmem_wait_ld();
        }
        if (lead) PATTN_K1_TRACE(30 + h);
        const int key0 = jt * kN;
        const int nvis = row_lim - key0;  // keys [key0, key0 + nvis) of this tile are visible
        if (cs < 0.f) {  // sign-adjust so that max(raw) * |c| = max(scaled)
#pragma unroll
          for (int c = 0; c < kN; ++c) s[c] = -s[c];
        }
        if (__any_sync(0xffffffffu, nvis < kN)) {  // diagonal / tail tile: causal mask (warp-uniform)
#pragma unroll
          for (int c = 0; c < kN; ++c) s[c] = c < nvis ? s[c] : -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = s[i];
#pragma unroll
        for (int c = 8; c < kN; ++c) mx[c & 7] = fmaxf(mx[c & 7], s[c]);
        const float mraw = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                           fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        if (lead) PATTN_K1_TRACE(32 + h);
        const float mt = mraw * ca;
        const float m_new = fmaxf(m_run, mt);
        float alpha = 1.f, m_use = m_run;
        if (m_new > m_run + kRescaleThreshold) {  // includes m_run == -inf
          alpha = fast_exp2(m_run - m_new);
          m_use = m_new;
        }
        const float nbase = m_use == -INFINITY ? 0.f : -m_use;
        // packed fp32x2 FMA-pipe ops (FFMA2 / FADD2, sm_100): half the instructions for the
        // exponent argument and the row sum
        const uint64_t ca2 = f32x2(ca, ca), nb2 = f32x2(nbase, nbase);
        uint64_t rs2[4] = {0ull, 0ull, 0ull, 0ull};
        uint32_t pk[kN / 2];
#pragma unroll
        for (int c = 0; c < kN; c += 2) {
          // e^{scale*qk - m} in the log2 domain
          const uint64_t xx = ffma2(f32x2(s[c], s[c + 1]), ca2, nb2);
          const float e0 = fast_exp2(f32x2_lo(xx)), e1 = fast_exp2(f32x2_hi(xx));
          rs2[(c >> 1) & 3] = fadd2(rs2[(c >> 1) & 3], f32x2(e0, e1));
          pk[c >> 1] = E::pack(e0, e1);
        }
        const uint64_t r01 = fadd2(rs2[0], rs2[1]), r23 = fadd2(rs2[2], rs2[3]), rr = fadd2(r01, r23);
        const float rs = f32x2_lo(rr) + f32x2_hi(rr);
        if (lead) PATTN_K1_TRACE(34 + h);
        // O_h: PV_h(jt-1) (issued once P_h(jt-1) arrived, while this tile's exponentials ran)
        // must be complete before O_h is corrected and before P_h(jt) can be consumed.
        // (the wait cannot be skipped when no row rescales: mbarrier parity only tells phases
        // apart one step back, so every pv_done phase must be observed in order)
        if (jt > 0) {
          mbar_wait(&bar.pv_done[h], (tc - 1) & 1u);
          tc_fence_after();
          // tcgen05.ld/st are warp-collective (.sync.aligned): rescale when ANY row of the warp needs it
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) {
              uint32_t o[32];
              PATTN_TMEM_LD32(tO + c0, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
              PATTN_TMEM_ST32(tO + c0, o);
            }
          }
        }
        l_run = l_run * alpha + rs;
        m_run = m_use;
        // P (bf16, 2 per column) over the first 32 columns of the S buffer: the A operand of PV_h
        PATTN_TMEM_ST32(tS + 0, (pk + 0));
        // Zero V rows of slots >= L inside the last fetched sub-block (they may hold NaN); each
        // warpgroup does it before releasing its own P (both write the same zeros).
        {
          const int z0 = x.L - key0, z1 = min(kN, nsb_valid * 16 - key0);
          if (z0 < z1 && z0 < kN) {
            const uint32_t s2 = vc % kVStages;
            mbar_wait(&bar.v_full[s2], (vc / kVStages) & 1u);
            uint8_t* vb = smem + kOffV + s2 * kTile;
            constexpr int kCh = D / 8;  // 16-byte chunks per V row
            for (int e = r; e < (z1 - z0) * kCh; e += kHalfM) {
              const int row = z0 + e / kCh, ch = e % kCh;
              *reinterpret_cast<uint4*>(vb + (row >> 3) * kGroup + (ch >> 3) * 1024 + (row & 7) * 128 + ((ch & 7) << 4)) =
                  make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();
          }
        }
        ++vc;
        tmem_wait_st();
        tc_fence_before();
        if (lead) PATTN_K1_TRACE(12 + h);
        mbar_arrive(&bar.p_full[h]);
        ++tc;
      }
      // ---- epilogue: O / l -> bf16 -> out (valid rows only)
      mbar_wait(&bar.pv_done[h], (tc - 1) & 1u);
      if (lead) PATTN_K1_TRACE(42 + h);
      tc_fence_after();
      // this warp's O columns in one go, then O_h is released to the next item's PV_h(0)
      // before the normalisation and the global stores
      uint32_t o[D];
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) PATTN_TMEM_LD32(tO + c0, (o + c0));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bar.o_empty[h]);
      // Full 8-token slices of a warp (32 rows, all valid) leave through a TMA store from a
      // 128B-swizzled staging slice: 8 STS.128 per thread and pass instead of 16 STG.128 that
      // each touch 32 different 128-B lines (rows are 256 B apart in `out`) -- those flooded
      // the MIO queue for ~4k clk per item and stalled the MMA warp's next S issue (trace).
      const int tk_last = h * bq_half + ((r | 31) / G);  // token of the warp's last row
      const bool tma_out = p.k1_tma_store && tk_last < x.ntok;
      uint8_t* stg0 = smem + kOffStage + (h * 4 + (warp & 3)) * kStageWarp;
      if (tma_out) {
        if (lane == 0) bulk_wait_group_read0();  // the slice's previous store has read it
        __syncwarp();
      }
      const float inv = 1.f / l_run;
      const uint64_t inv2 = f32x2(inv, inv);
      if (tma_out) {
        const uint32_t row_off = (uint32_t)(r & 31) * 128;
        const int tok_w = x.q0 + x.tok0 + h * bq_half + (r & ~31) / G;
#pragma unroll
        for (int pass = 0; pass < Sh::kHalves; ++pass) {
          uint8_t* stg = stg0 + pass * 4096;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int c0 = pass * 64 + c * 8;
            uint4 v;
            uint64_t a = fmul2((uint64_t)o[c0 + 0] | ((uint64_t)o[c0 + 1] << 32), inv2);
            v.x = E::pack(f32x2_lo(a), f32x2_hi(a));
            a = fmul2((uint64_t)o[c0 + 2] | ((uint64_t)o[c0 + 3] << 32), inv2);
            v.y = E::pack(f32x2_lo(a), f32x2_hi(a));
            a = fmul2((uint64_t)o[c0 + 4] | ((uint64_t)o[c0 + 5] << 32), inv2);
            v.z = E::pack(f32x2_lo(a), f32x2_hi(a));
            a = fmul2((uint64_t)o[c0 + 6] | ((uint64_t)o[c0 + 7] << 32), inv2);
            v.w = E::pack(f32x2_lo(a), f32x2_hi(a));
            *reinterpret_cast<uint4*>(stg + row_off + ((c ^ (r & 7)) << 4)) = v;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&tmO, stg, pass * 64, 0, x.kvh, tok_w);
            bulk_commit_group();
          }
        }
      } else if (row_valid) {
        OutT* orow = O + (int64_t)(x.q0 + x.tok0 + tk) * p.o_st_tok +
                              (int64_t)(x.kvh * G + (r % G)) * p.o_st_head;
#pragma unroll
        for (int c = 0; c < D; c += 8) {
          uint4 v;
          uint64_t a = fmul2((uint64_t)o[c + 0] | ((uint64_t)o[c + 1] << 32), inv2);
          v.x = E::pack(f32x2_lo(a), f32x2_hi(a));
          a = fmul2((uint64_t)o[c + 2] | ((uint64_t)o[c + 3] << 32), inv2);
          v.y = E::pack(f32x2_lo(a), f32x2_hi(a));
          a = fmul2((uint64_t)o[c + 4] | ((uint64_t)o[c + 5] << 32), inv2);
          v.z = E::pack(f32x2_lo(a), f32x2_hi(a));
          a = fmul2((uint64_t)o[c + 6] | ((uint64_t)o[c + 7] << 32), inv2);
          v.w = E::pack(f32x2_lo(a), f32x2_hi(a));
          *reinterpret_cast<uint4*>(orow + c) = v;
        }
      }
      if (lead) PATTN_K1_TRACE(44 + h);
    }
    if (lane == 0) bulk_wait_group0();  // epilogue stores complete before the CTA retires
    if (threadIdx.x == 128) PATTN_CTA_END(k1, ic);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace

bool prefill_supported(const Params& p) {
  if (getenv("PATTN_DISABLE_K1")) return false;
  // BLOCK_Q = 2 * floor(128 / G) tokens in two halves of 128 rows (padding rows when G does not
  // divide 128, e.g. G = 3, 5, 6, 7, 12); head_dim 64 or 128; block sizes that are not a
  // multiple of 16 take the gathered producers (16-byte aligned K/V rows)
  return (p.D == 64 || p.D == 128) && p.G >= 1 && p.G <= 64 && (p.bs % 16 == 0 || p.kv_vec16) &&
         p.Hkv <= kMaxKvHeadMaps;
}

int prefill_block_q(int G) { return 2 * (kHalfM / G); }

PrefillLaunch plan_prefill(const Params& p, int num_sms) {
  PrefillLaunch pl;
  pl.grid = num_sms;
  pl.smem = p.D == 64 ? K1Shape<64>::kSmemBytes : K1Shape<128>::kSmemBytes;
  return pl;
}

template <bool G>
static cudaError_t launch_prefill_g(const Params& p, const PrefillLaunch& pl, const CUtensorMap& tmQ,
                                    const CUtensorMap& tmO, const KvHeadMaps& kv, cudaStream_t stream) {
  auto kern = p.dtype == 2 ? (p.D == 64 ? k1_prefill<64, EltF16, G> : k1_prefill<128, EltF16, G>)
                           : (p.D == 64 ? k1_prefill<64, EltBf16, G> : k1_prefill<128, EltBf16, G>);
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), pl.smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3(pl.grid), dim3(kThreads), pl.smem, stream, tmQ, tmO, kv, p);
}

cudaError_t launch_prefill(const Params& p, const PrefillLaunch& pl, const CUtensorMap& tmQ, const CUtensorMap& tmO,
                           const KvHeadMaps& kv, cudaStream_t stream) {
  return p.bs % 16 == 0 ? launch_prefill_g<false>(p, pl, tmQ, tmO, kv, stream)
                        : launch_prefill_g<true>(p, pl, tmQ, tmO, kv, stream);
}

}  // namespace pattn
