// K6 -- paged KV write ("reshape and cache"): the step that fills the cache before the
// attention call.  The paper assumes it has happened ("Q, K, and V have already been
// computed ... and stored in the KV cache in blocks", §4.3; App. A);
// SPEC's write_kv op states the addressing:
//     pos  = ctx_b + i                      (token i of sequence b, ctx_b = L_b - q_b)
//     blk  = block_table[b][pos / bs] ;  slot = pos % bs
//     k_cache[blk][slot][h][:] = k_new[cu_b + i][h][:]   for every KV head h (same for V)
// A pure byte copy (bit-exact).  HBM-bound: 2 * T * Hkv * D * esz bytes read, the same
// written.  One warp per token (grid-stride over tokens): the token's sequence comes from
// a warp-cooperative search over cu_seqlens_q (32 entries per probe); its Hkv rows of
// D * esz bytes are moved as 16-byte vectors, lanes striding over (head, 16-B chunk) so a
// warp's loads and stores cover whole contiguous head rows (coalesced for any stride).
#include "common.cuh"
#include "kernels.h"

namespace pattn {
namespace {

// Last sequence b with cu[b] <= tok (cu non-decreasing, cu[0] = 0 <= tok < cu[B]).
// Warp-cooperative: each probe compares 32 entries, so B = 256 needs <= 2 probes.
__device__ __forceinline__ int find_seq(const int32_t* __restrict__ cu, int B, int tok, int lane) {
  int lo = 0, hi = B;  // answer in [lo, hi)
  while (hi - lo > 1) {
    const int n = hi - lo;
    const int step = (n + 31) / 32;
    const int idx = lo + lane * step;
    const bool le = idx < hi && __ldg(cu + idx) <= tok;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    const int last = 31 - __clz(m);  // lane 0 always satisfies cu[lo] <= tok
    lo = lo + last * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

__global__ void __launch_bounds__(256) k6_write_kv(WriteKvParams p) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int chunks_per_row = p.row_bytes >> 4;
  const int chunks = p.Hkv * chunks_per_row;
  for (int tok = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tok < p.T; tok += warps) {
    const int b = find_seq(p.cu_seqlens_q, p.B, tok, lane);
    const int cu_b = __ldg(p.cu_seqlens_q + b);
    const int q_b = __ldg(p.cu_seqlens_q + b + 1) - cu_b;
    const int pos = __ldg(p.seq_lens + b) - q_b + (tok - cu_b);
    const int blk = __ldg(p.block_table + (int64_t)b * p.bt_stride + pos / p.bs);
    const int slot = pos % p.bs;
    const char* ksrc = static_cast<const char*>(p.k_new) + (int64_t)tok * p.new_st_tok;
    const char* vsrc = static_cast<const char*>(p.v_new) + (int64_t)tok * p.new_st_tok;
    const int64_t dst_off = (int64_t)blk * p.kv_st_blk + (int64_t)slot * p.kv_st_tok;
    char* kdst = static_cast<char*>(p.k_cache) + dst_off;
    char* vdst = static_cast<char*>(p.v_cache) + dst_off;
    for (int c = lane; c < chunks; c += 32) {
      const int h = c / chunks_per_row, o = (c % chunks_per_row) << 4;
      const uint4 kv = __ldg(reinterpret_cast<const uint4*>(ksrc + h * p.new_st_head + o));
      const uint4 vv = __ldg(reinterpret_cast<const uint4*>(vsrc + h * p.new_st_head + o));
      *reinterpret_cast<uint4*>(kdst + h * p.kv_st_head + o) = kv;
      *reinterpret_cast<uint4*>(vdst + h * p.kv_st_head + o) = vv;
    }
  }
}

}  // namespace

cudaError_t launch_write_kv(const WriteKvParams& p, int num_sms, cudaStream_t stream) {
  if (p.T == 0) return cudaSuccess;
  const int warps_needed = p.T;
  int grid = (warps_needed + 7) / 8;
  grid = grid < num_sms * 8 ? grid : num_sms * 8;  // 8 warps/CTA, 8 CTAs/SM resident
  k6_write_kv<<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace pattn
