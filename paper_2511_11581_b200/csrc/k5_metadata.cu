// K5 -- device batch metadata (§6.1 "Computation of Metadata").
//
// From cu_seqlens_q and seq_lens (device-resident, no host sync) one CTA computes:
//   * per sequence b: q_b, L_b and its class -- "decode" (q_b == 1, routed to the
//     split-KV decode kernel K2 when decode_to_k2; reading R15) or "Q-block" (every
//     other non-empty sequence, routed to K1/K4);
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

constexpr int kThreads = 1024;

// Block-wide exclusive scan of one int per thread; returns the exclusive prefix and
// writes the block total to *total.
__device__ int block_exclusive_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < (kThreads >> 5)) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int warp_excl = warp ? s_warp[warp - 1] : 0;
  *total = s_warp[(kThreads >> 5) - 1];
  __syncthreads();
  return warp_excl + x - v;
}

__global__ void __launch_bounds__(kThreads) k5_metadata(Params p) {
  __shared__ int s_warp[32];
  __shared__ unsigned long long s_blocks;
  __shared__ int s_ndec;
  const int B = p.B;
  if (threadIdx.x == 0) {
    s_blocks = 0ull;
    s_ndec = 0;
  }
  __syncthreads();

  // pass 1: decode count and total decode KV blocks
  unsigned long long my_blocks = 0;
  int my_dec = 0;
  for (int b = threadIdx.x; b < B; b += kThreads) {
    int qb = p.cu_seqlens_q[b + 1] - p.cu_seqlens_q[b];
    if (p.decode_to_k2 && qb == 1) {
      my_dec += 1;
      my_blocks += (unsigned long long)((p.seq_lens[b] + p.bs - 1) / p.bs);
    }
  }
  if (my_dec) {
    atomicAdd(&s_ndec, my_dec);
    atomicAdd(&s_blocks, my_blocks);
  }
  __syncthreads();

  const long long units = (long long)p.Hkv * p.HG;
  long long C;
  if (p.split_mode == 1) {
    C = INT_MAX;
  } else {
    long long want = ((long long)s_blocks * units + p.target_items - 1) / p.target_items;
    C = want > p.min_chunk_blocks ? want : p.min_chunk_blocks;
    if (C < 1) C = 1;
  }

  // pass 2: scans
  int carry_qb = 0, carry_ch = 0;
  for (int base = 0; base < B; base += kThreads) {
    int b = base + threadIdx.x;
    int nqb = 0, nch = 0;
    if (b < B) {
      int qb = p.cu_seqlens_q[b + 1] - p.cu_seqlens_q[b];
      if (p.decode_to_k2 && qb == 1) {
        long long nblk = (p.seq_lens[b] + p.bs - 1) / p.bs;
        nch = (int)((nblk + C - 1) / C);
      } else if (qb > 0) {
        nqb = (qb + p.block_q - 1) / p.block_q;
      }
    }
    int tot_qb, tot_ch;
    int ex_qb = block_exclusive_scan(nqb, s_warp, &tot_qb);
    int ex_ch = block_exclusive_scan(nch, s_warp, &tot_ch);
    if (b < B) {
      p.cu_qb[b] = carry_qb + ex_qb;
      p.cu_ch[b] = carry_ch + ex_ch;
    }
    carry_qb += tot_qb;
    carry_ch += tot_ch;
  }
  if (threadIdx.x == 0) {
    p.cu_qb[B] = carry_qb;
    p.cu_ch[B] = carry_ch;
    p.hdr[kHdrTotalQBlocks] = carry_qb;
    p.hdr[kHdrNumDecodes] = s_ndec;
    p.hdr[kHdrTotalChunks] = carry_ch;
    p.hdr[kHdrBlockQ] = p.block_q;
    p.hdr[kHdrChunkBlocks] = (int)(C > INT_MAX ? INT_MAX : C);
    p.hdr[kHdrPrefillCounter] = 0;
    p.hdr[kHdrDecodeCounter] = 0;
  }
}

}  // namespace

cudaError_t launch_metadata(const Params& p, cudaStream_t stream) {
  k5_metadata<<<1, kThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace pattn
