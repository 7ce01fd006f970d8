// kernels.h -- host-callable launchers of the libpattn kernels (internal; not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "params.h"

namespace pattn {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size) instead of
// on every launch (pattn_api.cu).
cudaError_t ensure_dynamic_smem(const void* func, size_t bytes);

// Launch with programmatic stream serialization (PDL) unless PATTN_NO_PDL is set: the kernel
// may be scheduled while its stream predecessor finishes; it calls pdl_wait() before reading
// the predecessor's results.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  static const bool off = [] {
    const char* v = getenv("PATTN_NO_PDL");
    return v && *v && *v != '0';
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// K5: batch metadata + decode segment plan (one CTA).
cudaError_t launch_metadata(const Params& p, cudaStream_t stream);

// K4: generic SIMT Q-block kernel (fp32 / bf16, any q_len, any block size).
// rows_per_warp in {8, 16}: BLOCK_M = block_q * G <= 4 * rows_per_warp.
cudaError_t launch_generic(const Params& p, int grid, int rows_per_warp, cudaStream_t stream);
size_t generic_smem_bytes(const Params& p);

// K2: split-KV decode kernel (bf16, TMA-fed shared-memory ring, mma.sync dot products).
struct DecodeLaunch {
  int grid;
  int stages;
  int consumer_warps;
  size_t smem;
};
DecodeLaunch plan_decode(const Params& p, int num_sms, size_t max_smem, int ctas_per_sm);
cudaError_t launch_decode(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK, const CUtensorMap& tmV,
                          cudaStream_t stream);

// K2W: split-KV decode with head-wide TMA boxes (HB KV heads per request; k2w_decode.cu).
int wide_decode_heads(int Hkv, int G);  // HB in {8, 4, 2}, or 0 when K2W does not apply
DecodeLaunch plan_decode_wide(const Params& p, int num_sms, size_t max_smem);
cudaError_t launch_decode_wide(const Params& p, const DecodeLaunch& dl, const CUtensorMap& tmK,
                               const CUtensorMap& tmV, cudaStream_t stream);

// K3: segment reduction (LSE merge of decode partials).
cudaError_t launch_reduce(const Params& p, cudaStream_t stream);

// K1: tcgen05/TMEM prefill Q-block kernel (bf16, D = 128).
// Per-KV-head 5-D views of the K and V caches {64 d, 8 slots, 2 d-halves, bs/8 slot groups,
// block}, box {64, 8, 2, 2, 1}: one TMA box = one 16-key sub-block of one head, landing as
// [slot group][d half][8 slots][64 d] (4 KB), which UMMA reads with SBO = 2048.
constexpr int kMaxKvHeadMaps = 64;
struct KvHeadMaps {
  CUtensorMap k[kMaxKvHeadMaps];
  CUtensorMap v[kMaxKvHeadMaps];
};
struct PrefillLaunch {
  int grid;
  size_t smem;
};
bool prefill_supported(const Params& p);
int prefill_block_q(int G);  // tokens per K1 Q block (BLOCK_M / G)
PrefillLaunch plan_prefill(const Params& p, int num_sms);
cudaError_t launch_prefill(const Params& p, const PrefillLaunch& pl, const CUtensorMap& tmQ, const CUtensorMap& tmO,
                           const KvHeadMaps& kv, cudaStream_t stream);

// K7: the paper's baseline per-(token, head) kernel (App. A), PATTN_FLAG_BASELINE only.
cudaError_t launch_baseline(const Params& p, cudaStream_t stream);

// K6: paged KV write (reshape-and-cache).  Strides in BYTES; every row start and row_bytes
// are multiples of 16 (checked by the API).
struct WriteKvParams {
  const void* k_new;
  const void* v_new;
  void* k_cache;
  void* v_cache;
  const int32_t* block_table;
  const int32_t* cu_seqlens_q;
  const int32_t* seq_lens;
  int32_t B, T, Hkv, bs, row_bytes;
  int64_t new_st_tok, new_st_head;
  int64_t kv_st_blk, kv_st_tok, kv_st_head;
  int64_t bt_stride;  // elements
};
cudaError_t launch_write_kv(const WriteKvParams& p, int num_sms, cudaStream_t stream);

}  // namespace pattn
