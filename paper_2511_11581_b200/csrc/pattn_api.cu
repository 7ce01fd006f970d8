// pattn_api.cu -- the libpattn C ABI (include/pattn.h): validation, the host planner
// (H1: kernel routing, BLOCK_Q, segment policy, grids), TMA descriptors (H2) and the
// launch sequence K5 -> {K1 | K4} -> K2 -> K3 on the caller's stream(s).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <mutex>
#include <utility>
#include <vector>

#include "kernels.h"
#include "params.h"
#include "pattn.h"

using namespace pattn;

namespace {

constexpr int32_t kVersion = 100;  // 0.1.0

struct DeviceInfo {
  int sms = 0;
  size_t max_smem = 0;
  bool ok = false;
};

DeviceInfo device_info() {
  static std::mutex mu;
  static DeviceInfo cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return DeviceInfo{};
  std::lock_guard<std::mutex> g(mu);
  if (!cache[dev].ok) {
    int sms = 0, smem = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return DeviceInfo{};
    if (cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      return DeviceInfo{};
    cache[dev].sms = sms;
    cache[dev].max_smem = (size_t)smem;
    cache[dev].ok = true;
  }
  return cache[dev];
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool debug_sync() {
  static const bool on = [] {
    const char* v = getenv("PATTN_DEBUG_SYNC");
    return v && *v && *v != '0';
  }();
  return on;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

float env_float(const char* name, float dflt) {
  const char* v = getenv(name);
  return (v && *v) ? (float)atof(v) : dflt;
}

thread_local char g_last_error[256] = "";

pattn_status_t cuda_fail(cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return PATTN_ERR_CUDA;
}

}  // namespace

namespace pattn {
// Dynamic shared-memory opt-in, once per (kernel, device) and size (kernels.h).
cudaError_t ensure_dynamic_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  size_t& have = done[{func, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}
}  // namespace pattn

namespace {

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

// ---- tuning tree (pattn_set_tuning_tree): copied under a mutex, read by every plan
struct TuningTree {
  std::mutex mu;
  std::vector<pattn_tree_node_t> nodes;
};
TuningTree& tuning_tree() {
  static TuningTree t;
  return t;
}

bool leaf_ok(const pattn_tuning_t& t) {
  return t.items_per_sm >= 0 && t.items_per_sm <= 4096 && t.min_chunk_tokens >= 0 && t.min_chunk_tokens <= (1 << 24) &&
         t.decode_ctas_per_sm >= 0 && t.decode_ctas_per_sm <= 4 && t.k2_sm_mbs >= 0 && t.k2_sm_mbs <= 1000000 &&
         (t.serial == 0 || t.serial == 1) && t.decode_kernel >= 0 && t.decode_kernel <= 2;
}

double feature_value(const pattn_problem_t* p, int f) {
  switch (f) {
    case PATTN_FEAT_NUM_SEQS: return p->num_seqs;
    case PATTN_FEAT_NUM_TOKENS: return p->num_tokens;
    case PATTN_FEAT_MAX_QUERY_LEN: return p->max_query_len > 0 ? p->max_query_len : p->num_tokens;
    case PATTN_FEAT_MAX_SEQ_LEN:
      return p->max_seq_len > 0 ? p->max_seq_len : (double)p->max_blocks_per_seq * p->block_size;
  }
  return 0.0;
}

// Tree leaf for p (all zero when no tree is loaded), then env overrides, then defaults.
// *leaf_kernel: the decode kernel the leaf's decode knobs were measured with (before overrides).
pattn_tuning_t resolve_tuning(const pattn_problem_t* p, int* leaf_kernel = nullptr) {
  pattn_tuning_t t{0, 0, 0, 0, 0, 0};
  {
    TuningTree& tt = tuning_tree();
    std::lock_guard<std::mutex> g(tt.mu);
    if (!tt.nodes.empty()) {
      int i = 0;
      while (tt.nodes[i].feature >= 0) {
        const pattn_tree_node_t& n = tt.nodes[i];
        i = feature_value(p, n.feature) < n.threshold ? n.lt : n.ge;
      }
      t = tt.nodes[i].leaf;
    }
  }
  if (leaf_kernel) *leaf_kernel = t.decode_kernel == 2 ? 2 : 1;
  const char* e;
  if ((e = getenv("PATTN_ITEMS_PER_SM")) && *e) t.items_per_sm = atoi(e);
  if ((e = getenv("PATTN_MIN_CHUNK_TOKENS")) && *e) t.min_chunk_tokens = atoi(e);
  if ((e = getenv("PATTN_DECODE_CTAS")) && *e) t.decode_ctas_per_sm = atoi(e);
  if ((e = getenv("PATTN_K2_SM_GBS")) && *e) t.k2_sm_mbs = (int32_t)(atof(e) * 1000.0);
  if ((e = getenv("PATTN_SERIAL")) && *e) t.serial = atoi(e) ? 1 : 0;
  if ((e = getenv("PATTN_DECODE_WIDE")) && *e) t.decode_kernel = atoi(e) ? 1 : 2;
  if (t.decode_kernel <= 0) t.decode_kernel = 1;
  // items_per_sm and min_chunk_tokens stay 0 here: their defaults depend on the decode kernel
  // (make_plan: K2 16 items per SM and 256-key segments, K2W 2 and 128)
  if (t.decode_ctas_per_sm <= 0) t.decode_ctas_per_sm = 2;
  if (t.decode_ctas_per_sm > 4) t.decode_ctas_per_sm = 4;
  return t;
}

struct Plan {
  bool use_k1 = false, use_k2 = false, use_k4 = false, use_k7 = false;
  bool k4_decodes = false;  // decode segments on K4 (when K2 cannot take them)
  bool kv_vec16 = false;    // K/V rows 16-byte aligned (K4 vector loads)
  int block_q = 1, HG = 1, rpw = 8;
  int decode_hb = 0;  // > 0: decodes on K2W (head-wide boxes)
  int leaf_kernel = 1;  // the decode kernel the tuning leaf's decode knobs were measured with
  int decode_ctas = 2;  // K2 CTAs per SM
  bool use_leaf_rate = false;  // the partition model takes the leaf's / env's decode rate
  bool decode_gather = false;  // K2W with cp.async-gathered entries (block size not a multiple of 16)
  int target_items = 0, min_chunk = 1, split_mode = 0, max_chunks = 0;
  int num_sms = 148;
  size_t max_smem = 0;
  size_t off_hdr = 0, off_cuqb = 0, off_cuch = 0, off_pm = 0, off_pl = 0, off_pacc = 0, total = 0;
  int k4_grid = 1;
  DecodeLaunch dl{};
  PrefillLaunch pl{};
  bool kv_tok_inner = false;
  pattn_tuning_t tuning{};
};

pattn_status_t check_problem(const pattn_problem_t* p) {
  if (!p) return PATTN_ERR_INVALID_ARG;
  if (p->num_seqs <= 0) return PATTN_ERR_EMPTY_BATCH;
  if (p->num_tokens < 0 || p->num_q_heads <= 0 || p->num_kv_heads <= 0 || p->block_size <= 0 ||
      p->num_blocks <= 0 || p->max_blocks_per_seq <= 0)
    return PATTN_ERR_INVALID_ARG;
  if (p->num_q_heads % p->num_kv_heads != 0) return PATTN_ERR_INVALID_ARG;
  if (p->head_dim != 64 && p->head_dim != 128) return PATTN_ERR_UNSUPPORTED;
  if (p->dtype != PATTN_DTYPE_F32 && p->dtype != PATTN_DTYPE_BF16 && p->dtype != PATTN_DTYPE_F16)
    return PATTN_ERR_UNSUPPORTED;
  if (p->num_q_heads / p->num_kv_heads > 64) return PATTN_ERR_UNSUPPORTED;
  if (p->q_stride_tok <= 0 || p->q_stride_head <= 0 || p->kv_stride_blk <= 0 || p->kv_stride_tok <= 0 ||
      p->kv_stride_head <= 0 || p->bt_stride < p->max_blocks_per_seq || p->o_stride_tok <= 0 ||
      p->o_stride_head <= 0)
    return PATTN_ERR_INVALID_ARG;
  return PATTN_OK;
}

void fill_params(const pattn_problem_t* p, const Plan& pl, Params* k) {
  memset(k, 0, sizeof(*k));
  k->B = p->num_seqs;
  k->T = p->num_tokens;
  k->Hq = p->num_q_heads;
  k->Hkv = p->num_kv_heads;
  k->G = p->num_q_heads / p->num_kv_heads;
  k->D = p->head_dim;
  k->bs = p->block_size;
  k->num_blocks = p->num_blocks;
  k->dtype = p->dtype;
  k->block_q = pl.block_q;
  k->HG = pl.HG;
  k->decode_hb = pl.decode_hb;
  k->decode_gather = pl.decode_gather ? 1 : 0;
  k->max_chunks = pl.max_chunks;
  k->decode_split = (pl.use_k2 || pl.k4_decodes) ? 1 : 0;
  k->k4_decodes = pl.k4_decodes ? 1 : 0;
  k->kv_vec16 = pl.kv_vec16 ? 1 : 0;
  k->split_mode = pl.split_mode;
  k->target_items = pl.target_items;
  k->min_chunk_blocks = pl.min_chunk;
  k->num_sms = pl.num_sms;
  k->kv_tok_inner = pl.kv_tok_inner ? 1 : 0;
  k->q_st_tok = p->q_stride_tok;
  k->q_st_head = p->q_stride_head;
  k->kv_st_blk = p->kv_stride_blk;
  k->kv_st_tok = p->kv_stride_tok;
  k->kv_st_head = p->kv_stride_head;
  k->bt_stride = p->bt_stride;
  k->max_seq_len_hint = p->max_seq_len > 0 ? p->max_seq_len : p->max_blocks_per_seq * p->block_size;
  k->max_query_len_hint = p->max_query_len > 0 ? p->max_query_len : p->num_tokens;
  k->o_st_tok = p->o_stride_tok;
  k->o_st_head = p->o_stride_head;
}

// H1 planner.  Pure host arithmetic on host-visible sizes (no device reads).
pattn_status_t make_plan(const pattn_problem_t* p, const void* q, const void* kc, const void* vc, const void* out,
                         Plan* pl) {
  pattn_status_t st = check_problem(p);
  if (st != PATTN_OK) return st;
  DeviceInfo di = device_info();
  pl->tuning = resolve_tuning(p, &pl->leaf_kernel);
  pl->num_sms = di.ok ? di.sms : 148;
  pl->max_smem = di.ok ? di.max_smem : 227 * 1024;
  const int G = p->num_q_heads / p->num_kv_heads;
  const int D = p->head_dim;
  const bool bf16 = p->dtype == PATTN_DTYPE_BF16 || p->dtype == PATTN_DTYPE_F16;  // 16-bit: tensor-core paths
  const bool generic = (p->flags & PATTN_FLAG_FORCE_GENERIC) != 0;
  pl->HG = (G + 7) / 8;
  pl->kv_tok_inner = p->kv_stride_tok < p->kv_stride_head;

  // K2 (TMA ring) requirements: bf16, bs multiple of 16 (mma key tiles) and <= 256 (TMA box),
  // 16-byte aligned rows and strides, dense head_dim.
  const bool tma_ok = (p->kv_stride_blk % 8 == 0) && (p->kv_stride_tok % 8 == 0) && (p->kv_stride_head % 8 == 0) &&
                      (kc == nullptr || aligned16(kc)) && (vc == nullptr || aligned16(vc));
  const bool q_ok = (p->q_stride_tok % 8 == 0) && (p->q_stride_head % 8 == 0) && (q == nullptr || aligned16(q));
  const bool o_ok = (p->o_stride_tok % 8 == 0) && (p->o_stride_head % 8 == 0) && (out == nullptr || aligned16(out));
  pl->use_k2 = bf16 && !generic && p->block_size % 16 == 0 && tma_ok && q_ok && o_ok;
  // Block sizes that are not a multiple of 16 (no TMA box fits a page): decodes on K2W with
  // cp.async-gathered entries when its other conditions hold (G <= 16, 2 | Hkv, 16-byte rows)
  {
    const int64_t e2 = 2;
    const bool rows16 = (p->kv_stride_blk * e2) % 16 == 0 && (p->kv_stride_tok * e2) % 16 == 0 &&
                        (p->kv_stride_head * e2) % 16 == 0 && (kc == nullptr || aligned16(kc)) &&
                        (vc == nullptr || aligned16(vc));
    pl->decode_gather = bf16 && !generic && p->block_size % 16 != 0 && rows16 && q_ok && o_ok &&
                        pl->tuning.decode_kernel != 2 && wide_decode_heads(p->num_kv_heads, G) > 0;
    if (pl->decode_gather) pl->use_k2 = true;
  }
  if (p->flags & PATTN_FLAG_BASELINE) {  // the paper's baseline kernel alone (comparison only)
    pl->use_k7 = true;
    pl->use_k2 = false;
    pl->decode_gather = false;
  }

  // 16-byte aligned K/V rows: K4's vector loads, and the gathered K1 / K2W producers
  const int64_t esz = bf16 ? 2 : 4;
  pl->kv_vec16 = (p->kv_stride_blk * esz) % 16 == 0 && (p->kv_stride_tok * esz) % 16 == 0 &&
                 (p->kv_stride_head * esz) % 16 == 0 && (D * esz) % 16 == 0 && (kc == nullptr || aligned16(kc)) &&
                 (vc == nullptr || aligned16(vc));
  Params probe;
  fill_params(p, *pl, &probe);
  pl->use_k1 = bf16 && !generic && !pl->use_k7 && tma_ok && q_ok && o_ok && prefill_supported(probe);
  const int max_q = p->max_query_len > 0 ? p->max_query_len : p->num_tokens;
  const bool maybe_prefill = max_q > 1 || !pl->use_k2;
  if (pl->use_k1) {
    pl->block_q = prefill_block_q(G);  // BLOCK_M = 256 rows = BLOCK_Q tokens x G heads
    pl->use_k1 = maybe_prefill;
  } else {
    pl->block_q = G <= 32 ? std::max(1, 32 / G) : 1;
    pl->use_k4 = maybe_prefill && !pl->use_k7;
  }
  // No K2 (fp32, block sizes that are not a multiple of 16, unaligned strides): K4 runs the
  // decodes as split-KV segment units too (parallel tiled softmax on the SIMT path), merged by K3
  // (K3 stores 16-byte vectors: output rows must be 16-byte aligned, else decodes stay unsplit)
  const bool o_vec = (p->o_stride_tok * esz) % 16 == 0 && (p->o_stride_head * esz) % 16 == 0 &&
                     (out == nullptr || aligned16(out));
  pl->k4_decodes = !pl->use_k2 && !pl->use_k7 && o_vec;
  if (pl->k4_decodes) pl->use_k4 = true;
  const int bm = pl->block_q * G;
  pl->rpw = bm <= 32 ? 8 : 16;

  // Decode kernel.  K2W: decode items of HB KV heads (one TMA request per 16 keys x HB heads;
  // default whenever G <= 16 and 2 | Hkv, tuning decode_kernel 2 / PATTN_DECODE_WIDE=0 keeps K2).
  if (pl->use_k2 && pl->tuning.decode_kernel != 2) pl->decode_hb = wide_decode_heads(p->num_kv_heads, G);
  // Decode segment policy (parallel tiled softmax): target work items per SM and the
  // shortest segment.  The tuning leaf's values apply to the kernel it was measured with (its
  // decode_kernel); otherwise the kernel's defaults: K2 16 items per SM and 256-key segments; K2W,
  // whose items are HB x larger, 2 and 128 (the tuning sweep's best single configuration,
  // profiles/r02/tuning_holdout.json; more segments cost K3 partial traffic: config 4 at 32 per SM
  // wrote 153 MB of partials).
  // (environment overrides always apply)
  const bool leaf_fits = (pl->decode_hb > 0) == (pl->leaf_kernel == 1);
  auto env_set = [](const char* n) {
    const char* v = getenv(n);
    return v && *v;
  };
  const bool use_items = (leaf_fits || env_set("PATTN_ITEMS_PER_SM")) && pl->tuning.items_per_sm > 0;
  const bool use_min = (leaf_fits || env_set("PATTN_MIN_CHUNK_TOKENS")) && pl->tuning.min_chunk_tokens > 0;
  const bool use_ctas = leaf_fits || env_set("PATTN_DECODE_CTAS");
  const int items_per_sm = use_items ? pl->tuning.items_per_sm : (pl->decode_hb ? 2 : 16);
  const int min_tok = use_min ? pl->tuning.min_chunk_tokens : (pl->decode_hb ? 128 : 256);
  pl->decode_ctas = use_ctas ? pl->tuning.decode_ctas_per_sm : 2;
  pl->use_leaf_rate = (leaf_fits || env_set("PATTN_K2_SM_GBS")) && pl->tuning.k2_sm_mbs > 0;
  if (p->flags & PATTN_FLAG_NO_SPLIT) {
    pl->split_mode = 1;
    pl->target_items = 1;
    pl->min_chunk = 1;
  } else if (p->flags & PATTN_FLAG_FORCE_SPLIT) {
    pl->split_mode = 2;
    pl->target_items = pl->num_sms * 64;
    pl->min_chunk = 1;
  } else {
    pl->target_items = env_int("PATTN_TARGET_ITEMS", pl->num_sms * items_per_sm);
    pl->min_chunk = env_int("PATTN_MIN_CHUNK_BLOCKS", std::max(1, (min_tok + p->block_size - 1) / p->block_size));
  }
  if (pl->target_items < 1) pl->target_items = 1;
  if (pl->min_chunk < 1) pl->min_chunk = 1;
  const long long units = (long long)p->num_kv_heads * pl->HG;
  const long long seg_units = pl->k4_decodes  ? (long long)p->num_kv_heads  // K4: all G heads per item
                              : pl->decode_hb ? (long long)(p->num_kv_heads / pl->decode_hb)
                                              : units;
  pl->max_chunks = (pl->use_k2 || pl->k4_decodes)
                       ? (int)(p->num_seqs + (pl->target_items + seg_units - 1) / seg_units + 1)
                       : 0;

  // workspace layout
  size_t off = 0;
  pl->off_hdr = off;
  off = align256(off + kHdrWords * sizeof(int32_t));
  pl->off_cuqb = off;
  off = align256(off + (size_t)(p->num_seqs + 1) * sizeof(int32_t));
  pl->off_cuch = off;
  off = align256(off + (size_t)(p->num_seqs + 1) * sizeof(int32_t));
  const size_t rows = (size_t)pl->max_chunks * p->num_q_heads;
  pl->off_pm = off;
  off = align256(off + rows * sizeof(float));
  pl->off_pl = off;
  off = align256(off + rows * sizeof(float));
  pl->off_pacc = off;
  off = align256(off + rows * (size_t)D * sizeof(float));
  pl->total = off;

  // grids
  if (pl->use_k4) {
    const int ctas_per_sm = 4;
    const long long max_items = ((long long)std::max(1, p->num_tokens) + pl->max_chunks) * p->num_kv_heads;
    pl->k4_grid = (int)std::min<long long>(max_items, (long long)pl->num_sms * ctas_per_sm);
    if (pl->k4_grid < 1) pl->k4_grid = 1;
  }
  fill_params(p, *pl, &probe);
  if (pl->use_k2)
    pl->dl = pl->decode_hb ? plan_decode_wide(probe, pl->num_sms, pl->max_smem)
                           : plan_decode(probe, pl->num_sms, pl->max_smem, pl->decode_ctas);
  if (pl->use_k1) pl->pl = plan_prefill(probe, pl->num_sms);
  return PATTN_OK;
}

CUtensorMapDataType tma_dtype(const pattn_problem_t* p) {
  return p->dtype == PATTN_DTYPE_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
}

// H2: per-KV-head 5-D views for K1 {64 d, 8 slots, 2 d-halves, bs/8 slot groups, block}
// (the head is folded into the base address; strides deliberately not nested) so that one
// box {64, 8, 2, 2, 1} brings a 16-key sub-block in the [group][half][8][64] order UMMA
// reads with a uniform 2 KB stride between 8-key groups.  The maps of the last call are
// cached (the encode is ~1 us of host time per map).
bool encode_head_map(CUtensorMap* tm, const pattn_problem_t* p, const void* head_base) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[5] = {64, 8, (cuuint64_t)(p->head_dim / 64), (cuuint64_t)(p->block_size / 8),
                        (cuuint64_t)p->num_blocks};
  cuuint64_t strides[4] = {(cuuint64_t)p->kv_stride_tok * 2, 128, (cuuint64_t)p->kv_stride_tok * 2 * 8,
                           (cuuint64_t)p->kv_stride_blk * 2};
  cuuint32_t box[5] = {64, 8, (cuuint32_t)(p->head_dim / 64), 2, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(tm, tma_dtype(p), 5, const_cast<void*>(head_base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct HeadMapCache {
  std::mutex mu;
  bool valid = false;
  const void* k = nullptr;
  const void* v = nullptr;
  pattn_problem_t prob{};
  KvHeadMaps maps;
};

bool encode_head_maps(KvHeadMaps* out, const pattn_problem_t* p, const void* kc, const void* vc) {
  static HeadMapCache cache;
  std::lock_guard<std::mutex> lock(cache.mu);
  const bool hit = cache.valid && cache.k == kc && cache.v == vc && cache.prob.dtype == p->dtype &&
                   cache.prob.num_kv_heads == p->num_kv_heads &&
                   cache.prob.head_dim == p->head_dim && cache.prob.block_size == p->block_size &&
                   cache.prob.num_blocks == p->num_blocks && cache.prob.kv_stride_blk == p->kv_stride_blk &&
                   cache.prob.kv_stride_tok == p->kv_stride_tok && cache.prob.kv_stride_head == p->kv_stride_head;
  if (!hit) {
    cache.valid = false;
    for (int h = 0; h < p->num_kv_heads; ++h) {
      const int64_t off = (int64_t)h * p->kv_stride_head * 2;
      if (!encode_head_map(&cache.maps.k[h], p, static_cast<const uint8_t*>(kc) + off) ||
          !encode_head_map(&cache.maps.v[h], p, static_cast<const uint8_t*>(vc) + off))
        return false;
    }
    cache.k = kc;
    cache.v = vc;
    cache.prob = *p;
    cache.valid = true;
  }
  memcpy(out->k, cache.maps.k, sizeof(CUtensorMap) * p->num_kv_heads);
  memcpy(out->v, cache.maps.v, sizeof(CUtensorMap) * p->num_kv_heads);
  return true;
}

// H2b: 5-D view {64 d, slot, D/64 d-halves, head, block} (strides deliberately not nested:
// the d-half dim, 128 B, sits outside the slot dim) so that ONE box {64, 16, D/64, 1, 1}
// brings a whole 16-key sub-block of one head into shared memory as [half][slot][64 d],
// the layout two 4-D boxes give -- half the TMA issues for the decode producer.
bool encode_kv_map5(CUtensorMap* tm, const pattn_problem_t* p, const void* base, int box_heads = 1) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int halves = p->head_dim / 64;
  cuuint64_t dims[5] = {64, (cuuint64_t)p->block_size, (cuuint64_t)halves, (cuuint64_t)p->num_kv_heads,
                        (cuuint64_t)p->num_blocks};
  cuuint64_t strides[4] = {(cuuint64_t)p->kv_stride_tok * 2, 128, (cuuint64_t)p->kv_stride_head * 2,
                           (cuuint64_t)p->kv_stride_blk * 2};
  cuuint32_t box[5] = {64, 16, (cuuint32_t)halves, (cuuint32_t)box_heads, 1};  // K2W: HB heads per box
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(tm, tma_dtype(p), 5, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Q viewed as [T][Hkv][G][D]: box {64 d, G heads, BLOCK_Q tokens} -> BLOCK_M = BLOCK_Q*G rows
// of 128 B, token-major / head-minor (reading R8).
bool encode_q_map(CUtensorMap* tm, const pattn_problem_t* p, const void* q, int block_q) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int G = p->num_q_heads / p->num_kv_heads;
  cuuint64_t dims[4] = {(cuuint64_t)p->head_dim, (cuuint64_t)G, (cuuint64_t)p->num_kv_heads,
                        (cuuint64_t)std::max(1, p->num_tokens)};
  cuuint64_t strides[3] = {(cuuint64_t)p->q_stride_head * 2, (cuuint64_t)p->q_stride_head * 2 * G,
                           (cuuint64_t)p->q_stride_tok * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)G, 1, (cuuint32_t)(block_q / 2)};  // one 128-row half
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(tm, tma_dtype(p), 4, const_cast<void*>(q), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// out viewed like Q, [T][Hkv][G][D]: box {64 d, G heads, 1, 32/G tokens} = the 32 rows of one
// K1 epilogue warp (one 64-wide d half per store).  Needs 32 % G == 0.
bool encode_o_map(CUtensorMap* tm, const pattn_problem_t* p, void* out) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int G = p->num_q_heads / p->num_kv_heads;
  if (G > 32 || 32 % G != 0) return false;
  cuuint64_t dims[4] = {(cuuint64_t)p->head_dim, (cuuint64_t)G, (cuuint64_t)p->num_kv_heads,
                        (cuuint64_t)std::max(1, p->num_tokens)};
  cuuint64_t strides[3] = {(cuuint64_t)p->o_stride_head * 2, (cuuint64_t)p->o_stride_head * 2 * G,
                           (cuuint64_t)p->o_stride_tok * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)G, 1, (cuuint32_t)(32 / G)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(tm, tma_dtype(p), 4, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct EventRec {
  const pattn_exec_opts_t* o;
  cudaError_t rec(int idx, cudaStream_t s) const {
    if (o && o->events[idx]) return cudaEventRecord(static_cast<cudaEvent_t>(o->events[idx]), s);
    return cudaSuccess;
  }
};

// Fork/join events of the two-stream path, created once per (thread, device) and reused by
// every call of that thread (recording an event again is legal, also during graph capture).
struct ForkJoin {
  cudaEvent_t fork = nullptr, join = nullptr;
};
cudaError_t fork_join_events(ForkJoin* out) {
  static thread_local std::map<int, ForkJoin> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  ForkJoin& fj = cache[dev];
  if (!fj.fork && (e = cudaEventCreateWithFlags(&fj.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
  if (!fj.join && (e = cudaEventCreateWithFlags(&fj.join, cudaEventDisableTiming)) != cudaSuccess) return e;
  *out = fj;
  return cudaSuccess;
}

// Host-detectable argument errors of a call (before anything is enqueued).
pattn_status_t check_call(const pattn_problem_t* p, const Plan& pl, const void* q, const void* k_cache,
                          const void* v_cache, const int32_t* block_table, const int32_t* cu_seqlens_q,
                          const int32_t* seq_lens, float scale, const void* out, const void* workspace,
                          size_t workspace_bytes) {
  (void)p;
  if (!q || !k_cache || !v_cache || !block_table || !cu_seqlens_q || !seq_lens || !out || !workspace)
    return PATTN_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0) return PATTN_ERR_INVALID_ARG;
  if (workspace_bytes < pl.total) return PATTN_ERR_WORKSPACE_TOO_SMALL;
  if (!(scale == scale) || scale > 3.0e38f || scale < -3.0e38f) return PATTN_ERR_INVALID_ARG;
  return PATTN_OK;
}

pattn_status_t run(const pattn_problem_t* p, const void* q, const void* k_cache, const void* v_cache,
                   const int32_t* block_table, const int32_t* cu_seqlens_q, const int32_t* seq_lens, float scale,
                   void* out, void* workspace, size_t workspace_bytes, void* stream_v,
                   const pattn_exec_opts_t* opts, bool metadata_only) {
  Plan pl;
  pattn_status_t st = make_plan(p, q, k_cache, v_cache, out, &pl);
  if (st != PATTN_OK) return st;
  st = check_call(p, pl, q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, scale, out, workspace,
                  workspace_bytes);
  if (st != PATTN_OK) return st;

  cudaStream_t s1 = static_cast<cudaStream_t>(stream_v);
  cudaStream_t s2 = (opts && opts->stream2 && !(p->flags & PATTN_FLAG_SERIAL) && !pl.tuning.serial)
                        ? static_cast<cudaStream_t>(opts->stream2)
                        : s1;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  Params k;
  fill_params(p, pl, &k);
  k.q = q;
  k.k = k_cache;
  k.v = v_cache;
  k.out = out;
  k.block_table = block_table;
  k.cu_seqlens_q = cu_seqlens_q;
  k.seq_lens = seq_lens;
  k.scale = scale;
  k.scale_log2 = scale * 1.4426950408889634f;
  k.hdr = reinterpret_cast<int32_t*>(ws + pl.off_hdr);
  k.cu_qb = reinterpret_cast<int32_t*>(ws + pl.off_cuqb);
  k.cu_ch = reinterpret_cast<int32_t*>(ws + pl.off_cuch);
  k.part_m = reinterpret_cast<float*>(ws + pl.off_pm);
  k.part_l = reinterpret_cast<float*>(ws + pl.off_pl);
  k.part_acc = reinterpret_cast<float*>(ws + pl.off_pacc);

  CUtensorMap tmQ, tmO, tmK5, tmV5;
  memset(&tmO, 0, sizeof(tmO));
  static thread_local KvHeadMaps head_maps;  // 16 KB: kept off the stack
  if (!metadata_only) {
    if (pl.use_k2 && pl.decode_gather) {
      memset(&tmK5, 0, sizeof(tmK5));  // K2W gathers its entries with cp.async: no tensor maps
      memset(&tmV5, 0, sizeof(tmV5));
    } else if (pl.use_k2) {
      const int hb = pl.decode_hb > 0 ? pl.decode_hb : 1;
      if (!encode_kv_map5(&tmK5, p, k_cache, hb) || !encode_kv_map5(&tmV5, p, v_cache, hb)) return PATTN_ERR_UNSUPPORTED;
    }
    if (pl.use_k1 && p->block_size % 16 == 0) {  // (other block sizes: K1 gathers rows with cp.async)
      if (!encode_head_maps(&head_maps, p, k_cache, v_cache)) return PATTN_ERR_UNSUPPORTED;
    }
    if (pl.use_k1) {
      if (!encode_q_map(&tmQ, p, q, pl.block_q)) return PATTN_ERR_UNSUPPORTED;
      k.k1_tma_store = (!getenv("PATTN_K1_NO_TMA_STORE") && encode_o_map(&tmO, p, out)) ? 1 : 0;
    }
  }

  // K1 claim order for batches of equal Q-block counts: rank by rank within groups of sequences
  // holding this much K/V (c3p 8 x 8 MB: 286 -> 262 us serial; unbounded on c5's 32 x 8 MB lost
  // L2 reuse, 2541 -> 2840 us)
  k.k1_group_mb = env_int("PATTN_K1_GROUP_MB", 32);
  const bool two = !metadata_only && (s2 != s1) && pl.use_k2 && (pl.use_k1 || pl.use_k4);
  if (two && pl.use_k1) {
    // K1 and K2 run concurrently on disjoint SMs; K5 sizes the split from the batch with a
    // per-SM cost model of the two kernels (measured on B200)
    k.partition = 1;
    k.prefill_ctas_fixed = env_int("PATTN_PREFILL_SMS", 0);
    k.k1_tile_us = env_float("PATTN_K1_TILE_US", 2.2f);
    // per-SM decode rate of the partition model: the tree (if measured with this decode kernel) /
    // env value, else the measured default of the decode kernel in use (K2W: 100, K2: 61 GB/s/SM;
    // K2W swept 80 / 90 / 100 on configs 3 and 5: 362.5 / 359.5 / 358.1 us and 2653 / 2635 / 2643 us)
    k.k2_sm_gbs = pl.use_leaf_rate ? (float)pl.tuning.k2_sm_mbs * 1e-3f
                  : pl.decode_hb          ? env_float("PATTN_K2W_SM_GBS", 100.f)
                                          : 61.f;
    k.hbm_gbs = env_float("PATTN_HBM_GBS", 6300.f);
  }

  EventRec ev{opts};
  ForkJoin fj;
  if (two) {
    const cudaError_t e = fork_join_events(&fj);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  cudaError_t e = ev.rec(2 * PATTN_KERNEL_METADATA, s1);
  if (e == cudaSuccess) e = launch_metadata(k, s1);
  if (e == cudaSuccess) e = ev.rec(2 * PATTN_KERNEL_METADATA + 1, s1);
  if (e != cudaSuccess) return cuda_fail(e);
  if (metadata_only) return PATTN_OK;

  if (two) {
    e = cudaEventRecord(fj.fork, s1);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s2, fj.fork, 0);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  cudaStream_t sd = two ? s2 : s1;
  // Two streams: the prefill kernel is issued first so that its (one-per-SM) CTAs take
  // their SMs before the decode grid spreads over the GPU; the CTAs beyond K5's partition
  // exit at once, the decode CTAs fill those SMs and, claiming items dynamically, the SMs
  // the prefill CTAs release when they finish.  After the fork, every exit path records the
  // join so that stream2 is always joined back (a capture stays well formed).
  auto step = [&](int kind, cudaStream_t s, auto&& launch) {
    if (e != cudaSuccess) return;
    e = ev.rec(2 * kind, s);
    if (e == cudaSuccess) e = launch();
    if (e == cudaSuccess) e = ev.rec(2 * kind + 1, s);
  };
  if (pl.use_k1) step(PATTN_KERNEL_PREFILL, s1, [&] { return launch_prefill(k, pl.pl, tmQ, tmO, head_maps, s1); });
  if (pl.use_k2) {
    step(PATTN_KERNEL_DECODE, sd, [&] {
      return pl.decode_hb ? launch_decode_wide(k, pl.dl, tmK5, tmV5, sd) : launch_decode(k, pl.dl, tmK5, tmV5, sd);
    });
    step(PATTN_KERNEL_REDUCE, sd, [&] { return launch_reduce(k, sd); });
  }
  if (pl.use_k7) step(PATTN_KERNEL_BASELINE, s1, [&] { return launch_baseline(k, s1); });
  if (pl.use_k4) step(PATTN_KERNEL_GENERIC, s1, [&] { return launch_generic(k, pl.k4_grid, pl.rpw, s1); });
  if (pl.k4_decodes) step(PATTN_KERNEL_REDUCE, s1, [&] { return launch_reduce(k, s1); });
  if (two) {
    cudaError_t ej = cudaEventRecord(fj.join, s2);
    if (ej == cudaSuccess) ej = cudaStreamWaitEvent(s1, fj.join, 0);
    if (e == cudaSuccess) e = ej;
  }
  if (e != cudaSuccess) return cuda_fail(e);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (debug_sync() && cudaStreamIsCapturing(s1, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone) {
    // PATTN_DEBUG_SYNC=1: synchronise and check what the device saw against the host hints
    // (a max_query_len hint below the true maximum can drop the prefill kernel from the plan)
    int32_t viol = 0;
    e = cudaStreamSynchronize(s1);
    if (e == cudaSuccess) e = cudaMemcpy(&viol, k.hdr + kHdrHintViolation, sizeof(viol), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e);
    if (viol) {
      snprintf(g_last_error, sizeof(g_last_error), "a sequence's q_b exceeds the max_query_len hint");
      return PATTN_ERR_INVALID_SEQUENCE;
    }
  }
  return PATTN_OK;
}

}  // namespace

extern "C" {

size_t pattn_workspace_size(const pattn_problem_t* p) {
  Plan pl;
  if (make_plan(p, nullptr, nullptr, nullptr, nullptr, &pl) != PATTN_OK) return 0;
  return pl.total;
}

pattn_status_t pattn_unified_attention(const pattn_problem_t* p, const void* q, const void* k_cache,
                                       const void* v_cache, const int32_t* block_table,
                                       const int32_t* cu_seqlens_q, const int32_t* seq_lens, float scale,
                                       void* out, void* workspace, size_t workspace_bytes, void* stream) {
  return run(p, q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, scale, out, workspace, workspace_bytes,
             stream, nullptr, false);
}

pattn_status_t pattn_unified_attention_ex(const pattn_problem_t* p, const void* q, const void* k_cache,
                                          const void* v_cache, const int32_t* block_table,
                                          const int32_t* cu_seqlens_q, const int32_t* seq_lens, float scale,
                                          void* out, void* workspace, size_t workspace_bytes, void* stream,
                                          const pattn_exec_opts_t* opts) {
  return run(p, q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, scale, out, workspace, workspace_bytes,
             stream, opts, false);
}

// ---- end-to-end (host buffers) variant
namespace {
struct HostIoLayout {
  size_t base, q, bt, cu, sl, out, total;
};
bool hostio_layout(const pattn_problem_t* p, HostIoLayout* L) {
  size_t base = pattn_workspace_size(p);
  if (!base) return false;
  const size_t esz = p->dtype == PATTN_DTYPE_F32 ? 4 : 2;
  size_t off = align256(base);
  L->base = base;
  L->q = off;
  off = align256(off + (size_t)p->num_tokens * p->num_q_heads * p->head_dim * esz);
  L->bt = off;
  off = align256(off + (size_t)p->num_seqs * p->bt_stride * sizeof(int32_t));
  L->cu = off;
  off = align256(off + (size_t)(p->num_seqs + 1) * sizeof(int32_t));
  L->sl = off;
  off = align256(off + (size_t)p->num_seqs * sizeof(int32_t));
  L->out = off;
  off = align256(off + (size_t)p->num_tokens * p->num_q_heads * p->head_dim * esz);
  L->total = off;
  return true;
}
}  // namespace

size_t pattn_hostio_workspace_size(const pattn_problem_t* p) {
  HostIoLayout L;
  return hostio_layout(p, &L) ? L.total : 0;
}

pattn_status_t pattn_unified_attention_hostio(const pattn_problem_t* p, const void* q_host, const void* k_cache,
                                              const void* v_cache, const int32_t* block_table_host,
                                              const int32_t* cu_seqlens_q_host, const int32_t* seq_lens_host,
                                              float scale, void* out_host, void* workspace, size_t workspace_bytes,
                                              void* stream) {
  pattn_status_t st = check_problem(p);
  if (st != PATTN_OK) return st;
  if (!q_host || !block_table_host || !cu_seqlens_q_host || !seq_lens_host || !out_host || !workspace)
    return PATTN_ERR_INVALID_ARG;
  if (p->q_stride_head != p->head_dim || p->q_stride_tok != (int64_t)p->num_q_heads * p->head_dim ||
      p->o_stride_head != p->head_dim || p->o_stride_tok != (int64_t)p->num_q_heads * p->head_dim)
    return PATTN_ERR_INVALID_ARG;
  HostIoLayout L;
  if (!hostio_layout(p, &L)) return PATTN_ERR_INVALID_ARG;
  if (workspace_bytes < L.total) return PATTN_ERR_WORKSPACE_TOO_SMALL;
  {
    // everything run() checks on the host, checked before the copies are enqueued
    Plan pl;
    uint8_t* w8 = static_cast<uint8_t*>(workspace);
    st = make_plan(p, w8 + L.q, k_cache, v_cache, w8 + L.out, &pl);
    if (st == PATTN_OK)
      st = check_call(p, pl, w8 + L.q, k_cache, v_cache, reinterpret_cast<int32_t*>(w8 + L.bt),
                      reinterpret_cast<int32_t*>(w8 + L.cu), reinterpret_cast<int32_t*>(w8 + L.sl), scale, w8 + L.out,
                      workspace, L.base);
    if (st != PATTN_OK) return st;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const size_t esz = p->dtype == PATTN_DTYPE_F32 ? 4 : 2;
  const size_t qbytes = (size_t)p->num_tokens * p->num_q_heads * p->head_dim * esz;
  if (cudaMemcpyAsync(ws + L.q, q_host, qbytes, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(ws + L.bt, block_table_host, (size_t)p->num_seqs * p->bt_stride * 4, cudaMemcpyHostToDevice,
                      s) != cudaSuccess ||
      cudaMemcpyAsync(ws + L.cu, cu_seqlens_q_host, (size_t)(p->num_seqs + 1) * 4, cudaMemcpyHostToDevice, s) !=
          cudaSuccess ||
      cudaMemcpyAsync(ws + L.sl, seq_lens_host, (size_t)p->num_seqs * 4, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return PATTN_ERR_CUDA;
  st = run(p, ws + L.q, k_cache, v_cache, reinterpret_cast<int32_t*>(ws + L.bt), reinterpret_cast<int32_t*>(ws + L.cu),
           reinterpret_cast<int32_t*>(ws + L.sl), scale, ws + L.out, workspace, L.base, stream, nullptr, false);
  if (st != PATTN_OK) return st;
  if (cudaMemcpyAsync(out_host, ws + L.out, qbytes, cudaMemcpyDeviceToHost, s) != cudaSuccess) return PATTN_ERR_CUDA;
  return PATTN_OK;
}

const char* pattn_status_string(pattn_status_t s) {
  switch (s) {
    case PATTN_OK: return "PATTN_OK";
    case PATTN_ERR_INVALID_ARG: return "PATTN_ERR_INVALID_ARG";
    case PATTN_ERR_EMPTY_BATCH: return "PATTN_ERR_EMPTY_BATCH";
    case PATTN_ERR_INVALID_SEQUENCE: return "PATTN_ERR_INVALID_SEQUENCE";
    case PATTN_ERR_INDEX_OUT_OF_RANGE: return "PATTN_ERR_INDEX_OUT_OF_RANGE";
    case PATTN_ERR_UNSUPPORTED: return "PATTN_ERR_UNSUPPORTED";
    case PATTN_ERR_WORKSPACE_TOO_SMALL: return "PATTN_ERR_WORKSPACE_TOO_SMALL";
    case PATTN_ERR_CUDA: return "PATTN_ERR_CUDA";
  }
  return "PATTN_ERR_UNKNOWN";
}

pattn_status_t pattn_validate_metadata_host(const pattn_problem_t* p, const int32_t* cu, const int32_t* sl,
                                            const int32_t* bt) {
  if (!p) return PATTN_ERR_INVALID_ARG;
  if (p->num_seqs <= 0) return PATTN_ERR_EMPTY_BATCH;
  if (!cu || !sl || !bt || p->block_size <= 0) return PATTN_ERR_INVALID_ARG;
  if (cu[0] != 0 || cu[p->num_seqs] != p->num_tokens) return PATTN_ERR_INVALID_SEQUENCE;
  for (int b = 0; b < p->num_seqs; ++b) {
    const int64_t qb = (int64_t)cu[b + 1] - cu[b];
    if (qb < 0 || qb > sl[b]) return PATTN_ERR_INVALID_SEQUENCE;
    const int64_t nblk = ((int64_t)sl[b] + p->block_size - 1) / p->block_size;
    if (nblk > p->max_blocks_per_seq) return PATTN_ERR_INDEX_OUT_OF_RANGE;
    for (int64_t j = 0; j < nblk; ++j) {
      const int32_t id = bt[(int64_t)b * p->bt_stride + j];
      if (id < 0 || id >= p->num_blocks) return PATTN_ERR_INDEX_OUT_OF_RANGE;
    }
  }
  return PATTN_OK;
}

pattn_status_t pattn_debug_plan(const pattn_problem_t* p, const int32_t* cu_seqlens_q, const int32_t* seq_lens,
                                int32_t* plan_out, int32_t plan_capacity, void* workspace, size_t workspace_bytes,
                                void* stream) {
  if (!p || !plan_out || plan_capacity < 2 * p->num_seqs + 10) return PATTN_ERR_INVALID_ARG;
  Plan pl;
  pattn_status_t st = make_plan(p, nullptr, nullptr, nullptr, nullptr, &pl);
  if (st != PATTN_OK) return st;
  // metadata only: dummy non-null tensor pointers are never dereferenced by K5
  const void* dummy = workspace;
  st = run(p, dummy, dummy, dummy, cu_seqlens_q, cu_seqlens_q, seq_lens, 1.0f, workspace, workspace, workspace_bytes,
           stream, nullptr, true);
  if (st != PATTN_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const int B = p->num_seqs;
  if (cudaMemcpyAsync(plan_out, ws + pl.off_hdr, 8 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(plan_out + 8, ws + pl.off_cuqb, (B + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, s) !=
          cudaSuccess ||
      cudaMemcpyAsync(plan_out + 8 + B + 1, ws + pl.off_cuch, (B + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                      s) != cudaSuccess)
    return PATTN_ERR_CUDA;
  return PATTN_OK;
}

int32_t pattn_planned_launches(const pattn_problem_t* p) {
  Plan pl;
  if (make_plan(p, nullptr, nullptr, nullptr, nullptr, &pl) != PATTN_OK) return 0;
  return 1 + (pl.use_k1 ? 1 : 0) + (pl.use_k4 ? 1 : 0) + (pl.use_k7 ? 1 : 0) + (pl.use_k2 ? 2 : 0) +
         (pl.k4_decodes ? 1 : 0);
}

int32_t pattn_planned_kernels(const pattn_problem_t* p) {
  Plan pl;
  if (make_plan(p, nullptr, nullptr, nullptr, nullptr, &pl) != PATTN_OK) return 0;
  return (1 << PATTN_KERNEL_METADATA) | (pl.use_k1 ? 1 << PATTN_KERNEL_PREFILL : 0) |
         (pl.use_k2 ? (1 << PATTN_KERNEL_DECODE) | (1 << PATTN_KERNEL_REDUCE) : 0) |
         (pl.k4_decodes ? (1 << PATTN_KERNEL_REDUCE) : 0) |
         (pl.use_k4 ? 1 << PATTN_KERNEL_GENERIC : 0) | (pl.use_k7 ? 1 << PATTN_KERNEL_BASELINE : 0) |
         (pl.decode_hb ? PATTN_PLAN_DECODE_WIDE : 0);
}

pattn_status_t pattn_write_kv(const pattn_problem_t* p, const void* k_new, const void* v_new,
                              int64_t new_stride_tok, int64_t new_stride_head, void* k_cache, void* v_cache,
                              const int32_t* block_table, const int32_t* cu_seqlens_q, const int32_t* seq_lens,
                              void* stream) {
  if (!p) return PATTN_ERR_INVALID_ARG;
  if (p->num_seqs <= 0) return PATTN_ERR_EMPTY_BATCH;
  if (p->num_tokens < 0 || p->num_kv_heads <= 0 || p->block_size <= 0 || p->head_dim <= 0 ||
      p->max_blocks_per_seq <= 0 || p->bt_stride < p->max_blocks_per_seq || new_stride_tok <= 0 ||
      new_stride_head <= 0 || p->kv_stride_blk <= 0 || p->kv_stride_tok <= 0 || p->kv_stride_head <= 0)
    return PATTN_ERR_INVALID_ARG;
  if (p->dtype != PATTN_DTYPE_F32 && p->dtype != PATTN_DTYPE_BF16 && p->dtype != PATTN_DTYPE_F16)
    return PATTN_ERR_UNSUPPORTED;
  if (p->num_tokens == 0) return PATTN_OK;
  if (!k_new || !v_new || !k_cache || !v_cache || !block_table || !cu_seqlens_q || !seq_lens)
    return PATTN_ERR_INVALID_ARG;
  const int64_t esz = p->dtype == PATTN_DTYPE_F32 ? 4 : 2;
  WriteKvParams w{};
  w.k_new = k_new;
  w.v_new = v_new;
  w.k_cache = k_cache;
  w.v_cache = v_cache;
  w.block_table = block_table;
  w.cu_seqlens_q = cu_seqlens_q;
  w.seq_lens = seq_lens;
  w.B = p->num_seqs;
  w.T = p->num_tokens;
  w.Hkv = p->num_kv_heads;
  w.bs = p->block_size;
  w.row_bytes = (int32_t)(p->head_dim * esz);
  w.new_st_tok = new_stride_tok * esz;
  w.new_st_head = new_stride_head * esz;
  w.kv_st_blk = p->kv_stride_blk * esz;
  w.kv_st_tok = p->kv_stride_tok * esz;
  w.kv_st_head = p->kv_stride_head * esz;
  w.bt_stride = p->bt_stride;
  // 16-byte vector moves: every row start must be 16-B aligned
  if ((w.row_bytes | w.new_st_tok | w.new_st_head | w.kv_st_blk | w.kv_st_tok | w.kv_st_head) & 15 ||
      !aligned16(k_new) || !aligned16(v_new) || !aligned16(k_cache) || !aligned16(v_cache))
    return PATTN_ERR_UNSUPPORTED;
  const DeviceInfo di = device_info();
  if (!di.ok) return cuda_fail(cudaGetLastError());
  const cudaError_t e = launch_write_kv(w, di.sms, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PATTN_OK : cuda_fail(e);
}

pattn_status_t pattn_set_tuning_tree(const pattn_tree_node_t* nodes, int32_t n_nodes) {
  std::vector<pattn_tree_node_t> v;
  if (nodes && n_nodes > 0) {
    for (int i = 0; i < n_nodes; ++i) {
      const pattn_tree_node_t& n = nodes[i];
      if (n.feature < 0) {
        if (!leaf_ok(n.leaf)) return PATTN_ERR_INVALID_ARG;
      } else if (n.feature >= PATTN_FEAT_COUNT || n.lt <= i || n.ge <= i || n.lt >= n_nodes || n.ge >= n_nodes ||
                 !(n.threshold == n.threshold)) {
        return PATTN_ERR_INVALID_ARG;
      }
    }
    v.assign(nodes, nodes + n_nodes);
  }
  TuningTree& tt = tuning_tree();
  std::lock_guard<std::mutex> g(tt.mu);
  tt.nodes.swap(v);
  return PATTN_OK;
}

pattn_status_t pattn_plan_tuning(const pattn_problem_t* p, pattn_tuning_t* out) {
  if (!out) return PATTN_ERR_INVALID_ARG;
  const pattn_status_t st = check_problem(p);
  if (st != PATTN_OK) return st;
  *out = resolve_tuning(p);
  return PATTN_OK;
}

struct pattn_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

pattn_status_t pattn_graph_capture(const pattn_problem_t* p, const void* q, const void* k_cache, const void* v_cache,
                                   const int32_t* block_table, const int32_t* cu_seqlens_q, const int32_t* seq_lens,
                                   float scale, void* out, void* workspace, size_t workspace_bytes, void* stream,
                                   void* stream2, pattn_graph_t* graph) {
  if (!graph || !stream) return PATTN_ERR_INVALID_ARG;  // capture needs a real (non-legacy) stream
  *graph = nullptr;
  {
    // host-detectable errors first, before any capture is begun
    Plan pl;
    pattn_status_t st = make_plan(p, q, k_cache, v_cache, out, &pl);
    if (st == PATTN_OK)
      st = check_call(p, pl, q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, scale, out, workspace,
                      workspace_bytes);
    if (st != PATTN_OK) return st;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_fail(e);
  pattn_exec_opts_t o;
  memset(&o, 0, sizeof(o));
  o.stream2 = stream2;
  const pattn_status_t st = run(p, q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, scale, out, workspace,
                                workspace_bytes, stream, &o, false);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(s, &g);  // always end the capture, also after a failed enqueue
  if (st != PATTN_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (e != cudaSuccess) return cuda_fail(e);
  cudaGraphExec_t x = nullptr;
  e = cudaGraphInstantiateWithFlags(&x, g, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    return cuda_fail(e);
  }
  pattn_graph* h = new (std::nothrow) pattn_graph;
  if (!h) {
    cudaGraphExecDestroy(x);
    cudaGraphDestroy(g);
    return PATTN_ERR_INVALID_ARG;
  }
  h->graph = g;
  h->exec = x;
  *graph = h;
  return PATTN_OK;
}

pattn_status_t pattn_graph_launch(pattn_graph_t graph, void* stream) {
  if (!graph || !graph->exec) return PATTN_ERR_INVALID_ARG;
  const cudaError_t e = cudaGraphLaunch(graph->exec, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PATTN_OK : cuda_fail(e);
}

pattn_status_t pattn_graph_destroy(pattn_graph_t graph) {
  if (!graph) return PATTN_ERR_INVALID_ARG;
  cudaError_t e = cudaSuccess;
  if (graph->exec) e = cudaGraphExecDestroy(graph->exec);
  if (graph->graph) {
    const cudaError_t e2 = cudaGraphDestroy(graph->graph);
    if (e == cudaSuccess) e = e2;
  }
  delete graph;
  return e == cudaSuccess ? PATTN_OK : cuda_fail(e);
}

int32_t pattn_version(void) { return kVersion; }

const char* pattn_last_error(void) { return g_last_error; }

}  // extern "C"
