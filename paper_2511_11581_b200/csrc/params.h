// params.h -- kernel parameter block and workspace layout shared by the host planner
// (pattn_api.cu) and the kernels.  Plain C++ (no CUDA types) so the host side can
// include it anywhere.
#pragma once
#include <stdint.h>

namespace pattn {

// Workspace header (int32 words), written by the metadata kernel K5.
enum HdrWord {
  kHdrTotalQBlocks = 0,  // prefill Q blocks (sum over Q-block-kernel sequences)
  kHdrNumDecodes = 1,    // sequences routed to the decode kernel K2
  kHdrTotalChunks = 2,   // decode segments ("chunks") over all decode sequences
  kHdrBlockQ = 3,        // BLOCK_Q used for Q-block packing
  kHdrChunkBlocks = 4,   // decode segment length cap, in KV blocks
  kHdrPrefillCounter = 5,  // dynamic work counters (reset by K5)
  kHdrDecodeCounter = 6,
  kHdrPrefillCtas = 7,   // two-stream SM partition: K1 CTAs that work (the rest exit at once)
  kHdrHintViolation = 8, // K5: 1 if some q_b exceeds the max_query_len hint (the plan may miss it)
  kHdrDecodeClaimed = 9, // 1 once the decode kernel's item queue is empty (two-stream partition: K1
                         // CTAs that find their SM only after that may work on prefill items)
  kHdrQbUniform = 10,    // > 0: every Q-block sequence has this many Q blocks (K1 claims rank by rank)
  kHdrQbGroup = 11,      // with kHdrQbUniform: sequences per rank-by-rank claim group
  kHdrWords = 64
};

struct Params {
  // tensors
  const void* q;
  const void* k;
  const void* v;
  void* out;
  const int32_t* block_table;
  const int32_t* cu_seqlens_q;
  const int32_t* seq_lens;
  // sizes
  int32_t B, T, Hq, Hkv, G, D, bs, num_blocks;
  int32_t dtype;          // 0 fp32, 1 bf16 (pattn_dtype_t)
  int32_t block_q;        // query tokens per Q block
  int32_t HG;             // decode head groups of 8 per KV head = ceil(G/8)
  int32_t max_chunks;     // capacity of the partial buffers, in chunks
  int32_t decode_split;   // 1: q_b == 1 sequences are split-KV decode units (segments, K3 merge)
  int32_t k4_decodes;     // 1: those decode segments run on K4 (fp32 / block sizes K2 cannot fetch)
  int32_t kv_vec16;       // 1: K/V rows start 16-byte aligned (K4 loads them as 16-byte vectors)
  int32_t split_mode;     // 0 planner, 1 no split, 2 force split
  int32_t target_items;   // decode: desired number of (chunk, kv head, head group) items
  int32_t min_chunk_blocks;
  int32_t num_sms;
  int32_t decode_hb;      // > 0: decode on K2W, HB KV heads per TMA box / work item (Hkv / HB items per segment)
  int32_t decode_gather;  // K2W: 1 -> entries gathered row by row with cp.async (block size not a multiple of 16)
  int32_t kv_tok_inner;   // TMA dim order: 1 -> (d, slot, kvh, blk) [HND], 0 -> (d, kvh, slot, blk) [NHD]
  // Two-stream SM partition (K1 and K2 concurrent): K5 picks the number of SMs P for the
  // prefill kernel from the batch (cost model below); K1 CTAs >= P exit at once so that the
  // decode kernel's CTAs take those SMs.  partition 0: off (serial or single kernel).
  int32_t partition;
  int32_t prefill_ctas_fixed;  // > 0: use this P instead of the model (sweeps)
  float k1_tile_us;            // K1 cost per (128-key tile x 256-row Q block) on one SM
  int32_t k1_group_mb;         // K1 claim order: K/V megabytes per rank-by-rank sequence group
  float k2_sm_gbs;             // K2 K/V streaming rate of one SM (2 CTAs), GB/s
  float hbm_gbs;               // K2 ceiling: HBM read bandwidth, GB/s
  // strides (elements)
  int64_t q_st_tok, q_st_head;
  int64_t kv_st_blk, kv_st_tok, kv_st_head;
  int64_t bt_stride;
  int64_t o_st_tok, o_st_head;
  int32_t k1_tma_store;  // K1 epilogue: 1 -> full 8-token warp slices leave through a TMA store (tmO valid)
  float scale;       // softmax scale (Eq. 1)
  float scale_log2;  // scale * log2(e)
  // workspace
  int32_t* hdr;       // [kHdrWords]
  int32_t* cu_qb;     // [B+1]
  int32_t* cu_ch;     // [B+1]
  float* part_m;      // [max_chunks][Hq]   (log2 domain: max of scale*log2e*s)
  float* part_l;      // [max_chunks][Hq]
  float* part_acc;    // [max_chunks][Hq][D]
  int32_t max_seq_len_hint;    // host hint (max_seq_len, else max_blocks_per_seq * block_size)
  int32_t max_query_len_hint;  // host hint (max_query_len, else num_tokens); K5 flags q_b above it
};

}  // namespace pattn
