// K1 -- prefill / long-Q Q-block kernel on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// PAPER.md §4.4 "Prefill and GQA Optimization" (App. B): a Q block packs
// BLOCK_Q consecutive query tokens x the G query heads that share one KV head into a
// BLOCK_M = 128-row tile (token-major / head-minor, reading R8), so every K/V tile is
// loaded once per Q block and shared by all 128 rows.  KV tiles of 128 keys span
// 128/bs paged blocks (tile size decoupled from BLOCK_SIZE, §4.6); the tiled
// (online) softmax of §4.1 runs between the two contractions.
//
// One CTA per SM, persistent over (Q block, KV head) work items (static launch grid,
// P:401-406), longest (last) Q blocks first.  Warp roles (256 threads):
//   warp 0      TMA producer: Q tile (4-D map over q viewed [T][Hkv][G][D], 2 boxes),
//               K and V tiles (one 4-D box per paged block and 64-wide d half, through
//               the block table; blocks past the visible range are requested out of
//               bounds so TMA zero-fills them) into 2-stage K and V rings.
//   warp 1      MMA issuer (one thread): S = Q K^T (M=128, N=128, K=16 x 8) into a
//               double-buffered TMEM S tile; O += P V (P from shared memory, V MN-major)
//               into the TMEM O accumulator; tcgen05.commit -> mbarriers.
//   warp 2      TMEM allocator (512 columns: O | S0 | S1).
//   warps 4..7  softmax / correction / epilogue: thread r owns row r (TMEM lane r):
//               tcgen05.ld of the S row, causal mask (row limit ctx+i+1),
//               max, exp2, row sum; lazy rescale of O in TMEM only when the running
//               max grows by > 2^8 (exact: p <= 256 otherwise); P (bf16) written to
//               shared memory in the UMMA K-major SW128 layout; epilogue O / l -> bf16.
// V rows past the sequence end inside the last paged block may hold NaN (reading R13):
// the softmax warps zero them in shared memory before the PV product.
#include "common.cuh"
#include "kernels.h"

namespace pattn {
namespace {

constexpr int kM = 128;        // BLOCK_M rows per Q tile
constexpr int kN = 128;        // keys per KV tile
constexpr int kD = 128;        // head dim
constexpr int kThreads = 256;  // 8 warps
constexpr uint32_t kTile = kN * kD * 2;     // 32 KB: one bf16 128x128 tile
constexpr uint32_t kHalf = kTile / 2;       // 16 KB: one 64-wide d (or key) half
constexpr int kStages = 2;
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale O only if max grows by > 2^8

// shared-memory map (offsets from a 1024-aligned base)
constexpr uint32_t kOffQ = 0;
constexpr uint32_t kOffP = kOffQ + kTile;
constexpr uint32_t kOffK = kOffP + kTile;
constexpr uint32_t kOffV = kOffK + kStages * kTile;
constexpr uint32_t kOffBar = kOffV + kStages * kTile;
constexpr uint32_t kSmemBytes = kOffBar + 256 + 1024;

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], s_empty[2];
  uint64_t p_full, pv_done, o_empty;
  uint32_t tmem_base;
};

struct Item {
  int b, kvh, q0, qlen, L, ctx, tok0, ntok, kv_end, ntiles;
};

__device__ __forceinline__ Item prefill_item(const Params& p, int total_qb, int it) {
  Item x;
  const int j = total_qb - 1 - it / p.Hkv;  // last Q blocks (longest key range) first
  x.kvh = it % p.Hkv;
  x.b = upper_bound_minus1(p.cu_qb, p.B, j);  // App. B
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

__global__ void __launch_bounds__(kThreads, 1)
    k1_prefill(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars& bar = *reinterpret_cast<Bars*>(smem + kOffBar);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(&bar.q_full, 1);
    mbar_init(&bar.q_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.k_empty[s], 1);
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar.s_full[b], 1);
      mbar_init(&bar.s_empty[b], kM);
    }
    mbar_init(&bar.p_full, kM);
    mbar_init(&bar.pv_done, 1);
    mbar_init(&bar.o_empty, kM);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(&bar.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar.tmem_base;
  const uint32_t tmem_O = tmem;                   // columns [0, 128)
  const uint32_t tmem_S0 = tmem + 128;            // S buffer b at 128 + 128*b

  const int total_qb = p.hdr[kHdrTotalQBlocks];
  const int n_items = total_qb * p.Hkv;
  const int G = p.G;

  if (warp == 0) {
    // ================================================================ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
    }
    // A 128-key tile = 8 sub-blocks of 16 keys; sub-block i of tile jt is slots
    // [(idx % n16)*16, +16) of paged block bt[idx / n16], idx = 8*jt + i (any bs = 16k).
    constexpr int nbt = kN / 16;
    const int n16 = p.bs / 16;
    const uint64_t pol_kv = l2_policy_evict_last();  // K/V tiles are re-read by the sequence's other Q blocks
    uint32_t ic = 0, kc = 0, vc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++ic) {
      const Item x = prefill_item(p, total_qb, it);
      const int32_t* bt = p.block_table + (int64_t)x.b * p.bt_stride;
      const int nsb_valid = (x.kv_end + 15) / 16;  // sub-blocks holding visible keys
      if (lane == 0) {
        mbar_wait_tag(&bar.q_empty, (ic & 1u) ^ 1u, 1,(int)ic,it);
        mbar_arrive_expect_tx(&bar.q_full, kTile);
        tma_load_4d(smem + kOffQ, &tmQ, &bar.q_full, 0, 0, x.kvh, x.q0 + x.tok0);
        tma_load_4d(smem + kOffQ + kHalf, &tmQ, &bar.q_full, 64, 0, x.kvh, x.q0 + x.tok0);
      }
      // sub-blocks past the visible range are fetched at block index num_blocks: TMA zero-fills
      int id_next = (lane < nbt && lane < nsb_valid) ? __ldg(bt + lane / n16) : p.num_blocks;
      for (int jt = 0; jt < x.ntiles; ++jt) {
        const int id_cur = id_next;
        const int sb_next = (jt + 1) * nbt + lane;
        id_next = (jt + 1 < x.ntiles && lane < nbt && sb_next < nsb_valid) ? __ldg(bt + sb_next / n16) : p.num_blocks;
        // K tile
        {
          const uint32_t s = kc % kStages, ph = (kc / kStages) & 1u;
          if (lane == 0) {
            mbar_wait_tag(&bar.k_empty[s], ph ^ 1u, 2,(int)kc,it);
            mbar_arrive_expect_tx(&bar.k_full[s], kTile);
          }
          for (int i = 0; i < nbt; ++i) {
            const int blk = __shfl_sync(0xffffffffu, id_cur, i);
            const int slot0 = ((jt * nbt + i) % n16) * 16;
            const int c1 = p.kv_tok_inner ? slot0 : x.kvh, c2 = p.kv_tok_inner ? x.kvh : slot0;
            if (lane == 0) {
              uint8_t* dst = smem + kOffK + s * kTile + i * 16 * 128;
              tma_load_4d_hint(dst, &tmK, &bar.k_full[s], 0, c1, c2, blk, pol_kv);
              tma_load_4d_hint(dst + kHalf, &tmK, &bar.k_full[s], 64, c1, c2, blk, pol_kv);
            }
          }
          ++kc;
        }
        // V tile
        {
          const uint32_t s = vc % kStages, ph = (vc / kStages) & 1u;
          if (lane == 0) {
            mbar_wait_tag(&bar.v_empty[s], ph ^ 1u, 3,(int)vc,it);
            mbar_arrive_expect_tx(&bar.v_full[s], kTile);
          }
          for (int i = 0; i < nbt; ++i) {
            const int blk = __shfl_sync(0xffffffffu, id_cur, i);
            const int slot0 = ((jt * nbt + i) % n16) * 16;
            const int c1 = p.kv_tok_inner ? slot0 : x.kvh, c2 = p.kv_tok_inner ? x.kvh : slot0;
            if (lane == 0) {
              uint8_t* dst = smem + kOffV + s * kTile + i * 16 * 128;
              tma_load_4d_hint(dst, &tmV, &bar.v_full[s], 0, c1, c2, blk, pol_kv);
              tma_load_4d_hint(dst + kHalf, &tmV, &bar.v_full[s], 64, c1, c2, blk, pol_kv);
            }
          }
          ++vc;
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(kM, kN, 0, 0);   // Q (K-major) x K (K-major)
      constexpr uint32_t idPV = idesc_bf16_f32(kM, kD, 0, 1);  // P (K-major) x V (MN-major)
      uint32_t ic = 0, kc = 0, vc = 0, sc = 0, pc = 0;
      auto issue_pv = [&](int t) {
        mbar_wait_tag(&bar.p_full, pc & 1u, 11,(int)pc,t);
        const uint32_t s = vc % kStages, ph = (vc / kStages) & 1u;
        mbar_wait_tag(&bar.v_full[s], ph, 12,(int)vc,t);
        if (t == 0) mbar_wait_tag(&bar.o_empty, (ic & 1u) ^ 1u, 13,(int)ic,t);
        tc_fence_after();
        const uint32_t pa = sbase + kOffP, va = sbase + kOffV + s * kTile;
#pragma unroll
        for (int k = 0; k < kN / 16; ++k) {
          const uint64_t a = smem_desc_sw128(pa + (k >> 2) * kHalf + (k & 3) * 32, 16, 1024);
          const uint64_t bdesc = smem_desc_sw128(va + k * 2048, kHalf, 1024);
          tc_mma_f16_ss(tmem_O, a, bdesc, idPV, (t > 0 || k > 0) ? 1u : 0u);
        }
        tc_commit(&bar.pv_done);
        tc_commit(&bar.v_empty[s]);
        ++vc;
        ++pc;
      };
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++ic) {
        const Item x = prefill_item(p, total_qb, it);
        mbar_wait_tag(&bar.q_full, ic & 1u, 14,(int)ic,it);
        tc_fence_after();
        for (int jt = 0; jt < x.ntiles; ++jt) {
          const uint32_t s = kc % kStages, ph = (kc / kStages) & 1u;
          const uint32_t sb = sc & 1u, sph = (sc >> 1) & 1u;
          mbar_wait_tag(&bar.k_full[s], ph, 15,(int)kc,jt);
          mbar_wait_tag(&bar.s_empty[sb], sph ^ 1u, 16,(int)sc,jt);
          tc_fence_after();
          const uint32_t qa = sbase + kOffQ, ka = sbase + kOffK + s * kTile;
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint32_t off = (k >> 2) * kHalf + (k & 3) * 32;
            tc_mma_f16_ss(tmem_S0 + 128 * sb, smem_desc_sw128(qa + off, 16, 1024), smem_desc_sw128(ka + off, 16, 1024),
                          idS, k > 0 ? 1u : 0u);
          }
          tc_commit(&bar.s_full[sb]);
          tc_commit(&bar.k_empty[s]);
          if (jt == x.ntiles - 1) tc_commit(&bar.q_empty);
          ++kc;
          ++sc;
          if (jt > 0) issue_pv(jt - 1);
        }
        issue_pv(x.ntiles - 1);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ================================================================ softmax / correction / epilogue
    const int r = threadIdx.x - 128;  // row of the Q tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t pa = smem_u32(smem + kOffP);
    uint32_t sc = 0, pc = 0, vc = 0;
    __nv_bfloat16* O = static_cast<__nv_bfloat16*>(p.out);
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item x = prefill_item(p, total_qb, it);
      const int tk = r / G;
      const bool row_valid = tk < x.ntok;
      const int row_lim = min(x.ctx + x.tok0 + tk + 1, x.kv_end);  // keys [0, row_lim) visible
      const int nsb_valid = (x.kv_end + 15) / 16;  // 16-key sub-blocks fetched from the cache
      float m_run = -INFINITY, l_run = 0.f;
      for (int jt = 0; jt < x.ntiles; ++jt) {
        const uint32_t sb = sc & 1u, sph = (sc >> 1) & 1u;
        mbar_wait_tag(&bar.s_full[sb], sph, 21,(int)sc,jt);
        tc_fence_after();
        float s[kN];
        {
          uint32_t* su = reinterpret_cast<uint32_t*>(s);
          const uint32_t ta = tmem_S0 + 128 * sb + lane_off;
          PATTN_TMEM_LD32(ta + 0, (su + 0));
          PATTN_TMEM_LD32(ta + 32, (su + 32));
          PATTN_TMEM_LD32(ta + 64, (su + 64));
          PATTN_TMEM_LD32(ta + 96, (su + 96));
          tmem_wait_ld();
        }
        tc_fence_before();
        mbar_arrive(&bar.s_empty[sb]);
        ++sc;

        const int key0 = jt * kN;
        const int nvis = row_lim - key0;  // keys [key0, key0 + nvis) of this tile are visible
        float mt = -INFINITY;
#pragma unroll
        for (int c = 0; c < kN; ++c) {
          s[c] = c < nvis ? s[c] * p.scale_log2 : -INFINITY;
          mt = fmaxf(mt, s[c]);
        }
        const float m_new = fmaxf(m_run, mt);
        float alpha = 1.f, m_use = m_run;
        if (m_new > m_run + kRescaleThreshold) {  // includes m_run == -inf
          alpha = fast_exp2(m_run - m_new);
          m_use = m_new;
        }
        const float base = m_use == -INFINITY ? 0.f : m_use;
        float rs = 0.f;
#pragma unroll
        for (int c = 0; c < kN; ++c) {
          s[c] = fast_exp2(s[c] - base);
          rs += s[c];
        }
        // PV of the previous tile must be done before P (smem) and O (TMEM) are touched
        if (jt > 0) {
          mbar_wait_tag(&bar.pv_done, (pc - 1) & 1u, 22,(int)pc,jt);
          tc_fence_after();
          // tcgen05.ld/st are warp-collective (.sync.aligned): rescale when ANY row of the warp needs it
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
            for (int c0 = 0; c0 < kD; c0 += 32) {
              uint32_t o[32];
              PATTN_TMEM_LD32(tmem_O + lane_off + c0, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
              PATTN_TMEM_ST32(tmem_O + lane_off + c0, o);
            }
            tmem_wait_st();
          }
        }
        l_run = l_run * alpha + rs;
        m_run = m_use;
        // P row (bf16) -> shared memory, UMMA K-major SW128: [key half][row][128 B], chunk ^= row & 7
#pragma unroll
        for (int ch = 0; ch < kN / 8; ++ch) {
          uint4 v;
          v.x = pack_bf16(s[ch * 8 + 0], s[ch * 8 + 1]);
          v.y = pack_bf16(s[ch * 8 + 2], s[ch * 8 + 3]);
          v.z = pack_bf16(s[ch * 8 + 4], s[ch * 8 + 5]);
          v.w = pack_bf16(s[ch * 8 + 6], s[ch * 8 + 7]);
          const uint32_t addr = pa + (ch >> 3) * kHalf + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
                       "r"(v.w)
                       : "memory");
        }
        // zero V rows of slots >= L inside the last valid paged block (may hold NaN)
        const int z0 = x.L - key0, z1 = min(kN, nsb_valid * 16 - key0);
        if (z0 < z1 && z0 < kN) {
          const uint32_t s2 = vc % kStages, ph2 = (vc / kStages) & 1u;
          mbar_wait_tag(&bar.v_full[s2], ph2, 23,(int)vc,jt);
          uint8_t* vb = smem + kOffV + s2 * kTile;
          const int zs = max(z0, 0);
          for (int e = r; e < (z1 - zs) * 16; e += kM) {
            const int row = zs + (e >> 4), ch = e & 15;
            *reinterpret_cast<uint4*>(vb + (ch >> 3) * kHalf + row * 128 + ((ch & 7) << 4)) = make_uint4(0, 0, 0, 0);
          }
        }
        ++vc;
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bar.p_full);
        ++pc;
      }
      // ---- epilogue: O / l -> bf16 -> out (valid rows only)
      mbar_wait_tag(&bar.pv_done, (pc - 1) & 1u, 24,(int)pc,it);
      tc_fence_after();
      const float inv = 1.f / l_run;
      __nv_bfloat16* orow = O + (int64_t)(x.q0 + x.tok0 + tk) * p.o_st_tok + (int64_t)(x.kvh * G + (r - tk * G)) * p.o_st_head;
#pragma unroll
      for (int c0 = 0; c0 < kD; c0 += 32) {
        uint32_t o[32];
        PATTN_TMEM_LD32(tmem_O + lane_off + c0, o);
        tmem_wait_ld();
        if (row_valid) {
#pragma unroll
          for (int c = 0; c < 32; c += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(o[c + 0]) * inv, __uint_as_float(o[c + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(o[c + 2]) * inv, __uint_as_float(o[c + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(o[c + 4]) * inv, __uint_as_float(o[c + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(o[c + 6]) * inv, __uint_as_float(o[c + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + c0 + c) = v;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bar.o_empty);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace

bool prefill_supported(const Params& p) {
  if (getenv("PATTN_DISABLE_K1")) return false;
  return p.D == kD && p.G >= 1 && p.G <= kM && (kM % p.G) == 0 && p.bs % 16 == 0;
}

PrefillLaunch plan_prefill(const Params& p, int num_sms) {
  PrefillLaunch pl;
  pl.grid = num_sms;
  pl.smem = kSmemBytes;
  (void)p;
  return pl;
}

cudaError_t launch_prefill(const Params& p, const PrefillLaunch& pl, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                           const CUtensorMap& tmV, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(k1_prefill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
  if (e != cudaSuccess) return e;
  k1_prefill<<<pl.grid, kThreads, pl.smem, stream>>>(tmQ, tmK, tmV, p);
  return cudaGetLastError();
}

}  // namespace pattn
