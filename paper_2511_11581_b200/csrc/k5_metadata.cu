// K5 -- device batch metadata (§6.1 "Computation of Metadata").
//
// From cu_seqlens_q and seq_lens (device-resident, no host sync) one CTA computes:
//   * per sequence b: q_b, L_b and its class -- "decode" (q_b == 1: split-KV decode units
//     of K2, or of K4 for fp32 / block sizes K2 cannot fetch; reading R15) or "Q-block"
//     (every other non-empty sequence, routed to K1/K4);
//   * cu_q_blocks: exclusive scan of ceil(q_b / BLOCK_Q) over Q-block sequences
//      -- the total Q-block count is its last entry;
//   * the number of decodes and the decode segment plan: segment cap
//     C = max(min_chunk_blocks, ceil(total_decode_blocks * units / target_items)),
//     n_b = ceil(ceil(L_b/bs) / C) segments per decode sequence, cu_chunks = exclusive
//     scan of n_b.  Segments of a sequence are contiguous, equal-length (+-1 block)
//     ranges of KV blocks (parallel tiled softmax; reading R9).
//   * resets the dynamic work counters.
// Everything is integer arithmetic; results are bit-exact vs oracle/metadata.py.
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace pattn {

namespace {

constexpr int kMaxThreads = 1024;

// Block-wide sums of N unsigned 64-bit values per thread at once (all threads get the totals):
// one pair of barriers for all N (K5 is a single CTA on the critical path of every call).
template <int N>
__device__ void block_sum_u64(unsigned long long (&v)[N], unsigned long long (*s_red)[32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    if (lane == 0) s_red[i][warp] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    unsigned long long t = lane < nw ? s_red[i][lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    v[i] = t;
  }
  __syncthreads();
}

// K1 (Q block, 128-key tile) pairs of one Q-block sequence (the partition model's prefill work):
// sum over its Q blocks t0 = 0, bq, 2 bq, ... < qb of ceil((ctx + min(t0 + bq, qb)) / 128).
// K5 is one latency-bound warp chain per 32 sequences, so for BLOCK_Q a power of two <= 128 the
// sum runs over one period P = 128 / bq of the ceilings (term k + P = term k + 1) instead of
// every Q block; other BLOCK_Q walk the Q blocks.
__device__ __forceinline__ unsigned long long qblock_tiles(int ctx, int qb, int bq, int nqb) {
  unsigned long long s = (unsigned long long)((ctx + qb + 127) >> 7);  // the last (maybe short) Q block
  const int nf = nqb - 1;                                                // full ones end at ctx + k bq
  if (nf <= 0) return s;
  if (bq <= 128 && (bq & (bq - 1)) == 0) {
    const int lp = 7 - (31 - __clz(bq)), P = 1 << lp, m = nf >> lp, rem = nf - (m << lp);
    unsigned long long sp = 0, sr = 0;
    for (int r = 1; r <= P; ++r) {
      const unsigned long long f = (unsigned long long)((ctx + r * bq + 127) >> 7);
      sp += f;
      sr += r <= rem ? f : 0ull;
    }
    const unsigned long long mm = (unsigned long long)m;
    return s + mm * sp + (unsigned long long)P * (mm * (mm - 1) / 2) + sr + (unsigned long long)rem * mm;
  }
  for (int k = 1; k <= nf; ++k) s += (unsigned long long)((ctx + k * bq + 127) >> 7);
  return s;
}

// Block-wide exclusive scan of two ints per thread at once (x: Q blocks, y: decode
// segments); returns the exclusive prefixes and writes the block totals.
__device__ int2 block_exclusive_scan2(int2 v, int2* s_warp, int2* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int2 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, x.x, o), b = __shfl_up_sync(0xffffffffu, x.y, o);
    if (lane >= o) {
      x.x += a;
      x.y += b;
    }
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int2 w = lane < nw ? s_warp[lane] : make_int2(0, 0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, w.x, o), b = __shfl_up_sync(0xffffffffu, w.y, o);
      if (lane >= o) {
        w.x += a;
        w.y += b;
      }
    }
    s_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const int2 we = warp ? s_warp[warp - 1] : make_int2(0, 0);
  *total = s_warp[nw - 1];
  __syncthreads();
  return make_int2(we.x + x.x - v.x, we.y + x.y - v.y);
}

// One CTA of min(1024, roundup(B, 32)) threads; sequence b is handled by thread b % blockDim
// (one pass over the batch when B <= blockDim: per-sequence values stay in registers).
__global__ void __launch_bounds__(kMaxThreads) k5_metadata(Params p) {
  pdl_trigger();  // the next kernel may be scheduled now; it waits for this grid (pdl_wait)
  __shared__ unsigned long long s_red[9][32];
  __shared__ int2 s_scan[32];
  const int B = p.B;
  const int nt = blockDim.x;
  const bool one_pass = B <= nt;

  // pass 1: decode count and total decode KV blocks (+ the partition cost model's inputs:
  // K1 (Q block, 128-key tile) pairs and decode keys)
  int q0 = 0, L0 = 0, nqb0 = 0;  // this thread's sequence when one_pass (q_b, L_b, Q blocks)
  unsigned long long my_blocks = 0, my_tiles = 0, my_keys = 0, my_dec = 0, my_viol = 0;
  // Q-block sequences: count, sum of their Q blocks, of squares, of their keys
  unsigned long long my_qs = 0, my_nqb = 0, my_nqb2 = 0, my_qkeys = 0;
  for (int b = threadIdx.x; b < B; b += nt) {
    const int qb = __ldg(p.cu_seqlens_q + b + 1) - __ldg(p.cu_seqlens_q + b);
    const int L = __ldg(p.seq_lens + b);
    q0 = qb;
    L0 = L;
    my_viol += qb > p.max_query_len_hint ? 1ull : 0ull;  // the host planned with a smaller bound
    if (p.decode_split && qb == 1) {
      my_dec += 1;
      my_blocks += (unsigned long long)((L + p.bs - 1) / p.bs);
      my_keys += (unsigned long long)L;
    } else if (qb > 0) {
      nqb0 = (qb + p.block_q - 1) / p.block_q;
      const unsigned long long nqb = (unsigned long long)nqb0;
      my_qs += 1;
      my_nqb += nqb;
      my_nqb2 += nqb * nqb;
      my_qkeys += (unsigned long long)L;
      if (p.partition) my_tiles += qblock_tiles(L - qb, qb, p.block_q, nqb0);
    }
  }
  unsigned long long sums[9] = {my_dec, my_viol, my_blocks, my_tiles, my_keys, my_qs, my_nqb, my_nqb2, my_qkeys};
  block_sum_u64<9>(sums, s_red);
  const unsigned long long n_dec = sums[0], n_viol = sums[1], dec_blocks = sums[2];
  const unsigned long long tiles = p.partition ? sums[3] : 0ull, keys = p.partition ? sums[4] : 0ull;
  // Every Q-block sequence has the same number of Q blocks (sum of squares x count == square of
  // the sum) -> K1 claims its items rank by rank across a group of sequences (the r-th last Q
  // block of each before any (r+1)-th last): longest first within the group.  Groups hold as
  // many sequences as fit k1_group_mb of K/V (L2 reuse: all Q blocks of a sequence read its K/V).
  const unsigned long long n_qs = sums[5], s_nqb = sums[6], s_nqb2 = sums[7], s_qkeys = sums[8];
  // (32-bit and float arithmetic: the counts fit, and the group size is a heuristic)
  const int qb_uniform = (n_qs > 0 && s_nqb2 * n_qs == s_nqb * s_nqb) ? (int)((unsigned)s_nqb / (unsigned)n_qs) : 0;
  int qb_group = 1;
  if (qb_uniform > 0) {
    const float seq_bytes = (float)s_qkeys * (float)(p.Hkv * p.D * 2 * (p.dtype == 0 ? 4 : 2));  // x n_qs
    const float g = __fdividef((float)p.k1_group_mb * 1048576.f * (float)n_qs, fmaxf(seq_bytes, 1.f));
    qb_group = g >= (float)n_qs ? (int)n_qs : max(1, (int)g);
  }

  // SM partition for concurrent K1 / K2: P minimising max(prefill time on P SMs, decode
  // time on the other SMs, capped by HBM), from per-SM rates of the two kernels.
  int P = p.num_sms;
  if (p.partition) {
    if (p.prefill_ctas_fixed > 0) {
      P = min(p.prefill_ctas_fixed, p.num_sms);
    } else if (tiles > 0 && keys > 0) {
      // prefill time tp / c on c SMs; decode time bytes / min((S - c) b, HBM).  Balance
      // point c* = S tp b / (tp b + bytes); below c_hbm = S - HBM / b the decode side is
      // HBM-bound anyway, so P = max(c*, c_hbm).
      const float S = (float)p.num_sms;
      const float tp = (float)tiles * (float)p.Hkv * p.k1_tile_us * 1e-6f;  // SM-s
      const float bytes = (float)keys * (float)p.Hkv * (float)p.D * 4.0f;   // K + V bf16
      const float b = p.k2_sm_gbs * 1e9f;                                   // B/s per SM
      const float cstar = S * tp * b / (tp * b + bytes);
      const float chbm = S - p.hbm_gbs / p.k2_sm_gbs;
      P = (int)(fmaxf(cstar, chbm) + 0.5f);
      P = max(1, min(P, p.num_sms - 1));
    }
  }
  const long long target = p.target_items;
  const long long units = p.k4_decodes    ? (long long)p.Hkv
                          : p.decode_hb ? (long long)(p.Hkv / p.decode_hb)
                                        : (long long)p.Hkv * p.HG;  // items per segment
  long long C;
  if (p.split_mode == 1) {
    C = INT_MAX;
  } else {
    long long want = ((long long)dec_blocks * units + target - 1) / target;
    C = want > p.min_chunk_blocks ? want : p.min_chunk_blocks;
    if (C < 1) C = 1;
  }

  // pass 2: scans of Q blocks (cu_q_blocks) and decode segments (cu_chunks)
  int carry_qb = 0, carry_ch = 0;
  for (int base = 0; base < B; base += nt) {
    const int b = base + threadIdx.x;
    int2 cnt = make_int2(0, 0);
    if (b < B) {
      int qb = q0, L = L0;
      if (!one_pass) {
        qb = __ldg(p.cu_seqlens_q + b + 1) - __ldg(p.cu_seqlens_q + b);
        L = __ldg(p.seq_lens + b);
      }
      if (p.decode_split && qb == 1) {
        const long long nblk = (L + p.bs - 1) / p.bs;
        cnt.y = (int)((nblk + C - 1) / C);
      } else if (qb > 0) {
        cnt.x = one_pass ? nqb0 : (qb + p.block_q - 1) / p.block_q;
      }
    }
    int2 tot;
    const int2 ex = block_exclusive_scan2(cnt, s_scan, &tot);
    if (b < B) {
      p.cu_qb[b] = carry_qb + ex.x;
      p.cu_ch[b] = carry_ch + ex.y;
    }
    carry_qb += tot.x;
    carry_ch += tot.y;
  }
  if (threadIdx.x == 0) {
    p.cu_qb[B] = carry_qb;
    p.cu_ch[B] = carry_ch;
    p.hdr[kHdrTotalQBlocks] = carry_qb;
    p.hdr[kHdrNumDecodes] = (int)n_dec;
    p.hdr[kHdrTotalChunks] = carry_ch;
    p.hdr[kHdrBlockQ] = p.block_q;
    p.hdr[kHdrChunkBlocks] = (int)(C > INT_MAX ? INT_MAX : C);
    p.hdr[kHdrPrefillCounter] = 0;
    p.hdr[kHdrDecodeCounter] = 0;
    p.hdr[kHdrHintViolation] = n_viol ? 1 : 0;
    p.hdr[kHdrDecodeClaimed] = 0;
    p.hdr[kHdrQbUniform] = qb_uniform;
    p.hdr[kHdrQbGroup] = qb_group;
    p.hdr[kHdrPrefillCtas] = P;
  }
}

}  // namespace

cudaError_t launch_metadata(const Params& p, cudaStream_t stream) {
  const int threads = p.B >= kMaxThreads ? kMaxThreads : ((p.B + 31) / 32) * 32;
  k5_metadata<<<1, threads < 32 ? 32 : threads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace pattn
