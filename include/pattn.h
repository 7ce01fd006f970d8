/*
 * include/pattn.h -- libpattn: B200-native unified paged attention (C ABI).
 *
 * One call computes attention for a mixed batch of prefill, chunked-prefill and
 * decode sequences over a vLLM-style paged KV cache, as stated by
 * arXiv 2511.11581 ("The Anatomy of a Triton Attention Kernel"):
 *
 *   - Q, K and V are already computed; K/V of ALL tokens, including the current
 *     query tokens, are already stored in the paged KV cache (App. A
 *     P:10-11, §4.3).
 *   - The cache is addressed through a block table; BLOCK_SIZE = tokens per
 *     block (App. A, §4.3).
 *   - Per sequence b: query length q_b = cu_seqlens_q[b+1] - cu_seqlens_q[b]
 *     (accumulated query lengths, App. A), sequence length
 *     L_b = seq_lens[b] = context + query (§4.2), context
 *     ctx_b = L_b - q_b.  Query row i of b attends to keys
 *     0 .. ctx_b + i (self-inclusive prefix; R1/R2).
 *   - out[tok][h] = softmax(scale * q[tok][h] . K^T) V  (Eq. 1 P:212-216,
 *     stable softmax Eq. 2) with K/V taken from KV head
 *     h / (Hq/Hkv) (GQA, §4.1; R3).
 *
 * Conventions (all functions):
 *   - Device pointers are CUDA device pointers owned by the caller; the library
 *     never allocates device memory and never frees caller memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Asynchronous: the device work is enqueued on `stream`; the call returns
 *     without synchronising and performs NO device->host copies.  The caller
 *     synchronises before reading `out`.
 *   - Errors detectable on the host (null pointers, inconsistent sizes, an
 *     unsupported head_dim/dtype, too small a workspace) are returned before
 *     anything is enqueued.  Device-resident metadata (cu_seqlens_q, seq_lens,
 *     block_table) is TRUSTED on the hot path: violations are detected only by
 *     pattn_validate_metadata_host().  CUDA launch failures return
 *     PATTN_ERR_CUDA.
 *   - Thread safety: concurrent calls are safe when they use distinct
 *     workspaces.  The library caches only immutable per-device data.
 *   - q_b = 0 sequences are legal (padding) and produce no rows.
 *   - Host hints (pattn_problem_t.max_query_len / max_seq_len) must be upper bounds.  A
 *     max_query_len below the true maximum can drop the Q-block kernel from the plan; the
 *     metadata kernel flags it in the workspace, and with the environment variable
 *     PATTN_DEBUG_SYNC=1 every call synchronises its stream and returns
 *     PATTN_ERR_INVALID_SEQUENCE in that case (debugging aid; not for the hot path, and
 *     skipped while the stream is being captured into a CUDA graph).
 *   - Environment overrides of the planner (sweeps and A/B only): PATTN_ITEMS_PER_SM,
 *     PATTN_MIN_CHUNK_TOKENS, PATTN_DECODE_CTAS, PATTN_K2_SM_GBS, PATTN_SERIAL,
 *     PATTN_DECODE_WIDE (1 / 0 = decode_kernel 1 / 2) (see pattn_tuning_t),
 *     PATTN_PREFILL_SMS (fixed two-stream split), PATTN_DISABLE_K1, PATTN_DECODE_WIDE_HB
 *     (cap on K2W's heads per box), PATTN_K2W_SM_GBS (the partition model's K2W rate),
 *     PATTN_DECODE_SMS / PATTN_DECODE_RING_KB (decode grid and ring size, for sweeps),
 *     PATTN_TARGET_ITEMS / PATTN_MIN_CHUNK_BLOCKS (segment plan), PATTN_NO_PDL,
 *     PATTN_K1_TILE_US (the partition model's K1 cost per tile), PATTN_K1_GROUP_MB (K1's
 *     claim groups for batches of equal Q-block counts; results do not depend on it).
 */
#ifndef PATTN_H_
#define PATTN_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PATTN_API __attribute__((visibility("default")))
#else
#define PATTN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pattn_status {
  PATTN_OK = 0,
  PATTN_ERR_INVALID_ARG = 1,         /* bad sizes/strides/pointers (SPEC ShapeError/InvalidConfig) */
  PATTN_ERR_EMPTY_BATCH = 2,         /* num_seqs == 0 (SPEC EmptyBatch S:59) */
  PATTN_ERR_INVALID_SEQUENCE = 3,    /* q_b < 0, q_b > L_b, cu_seqlens_q[0] != 0 */
  PATTN_ERR_INDEX_OUT_OF_RANGE = 4,  /* block id outside [0, num_blocks) or table too short */
  PATTN_ERR_UNSUPPORTED = 5,         /* head_dim / dtype / alignment the kernels do not implement */
  PATTN_ERR_WORKSPACE_TOO_SMALL = 6,
  PATTN_ERR_CUDA = 7
} pattn_status_t;

typedef enum pattn_dtype {
  PATTN_DTYPE_F32 = 0,  /* q, caches and out are fp32; exact-ish SIMT path (tol 1e-5) */
  PATTN_DTYPE_BF16 = 1, /* q, caches and out are bf16; fp32 accumulation (tol 1e-2 abs + 1e-2 rel) */
  PATTN_DTYPE_F16 = 2   /* q, caches and out are fp16; the bf16 paths with fp16 storage (same tolerance) */
} pattn_dtype_t;

/*
 * Problem description.  Sizes are host-known from tensor shapes; the two
 * max_* fields are host HINTS (upper bounds) used only to size grids and the
 * workspace -- a hint smaller than the true value is an error the library does
 * not detect.  All strides are in ELEMENTS; the innermost (head_dim) stride of
 * q, the caches and out must be 1 and every row must be 16-byte aligned.
 *
 *   q        [num_tokens][num_q_heads][head_dim]       strides (q_stride_tok, q_stride_head, 1)
 *   k_cache, v_cache: element (blk, slot, kvh, d) at
 *            blk*kv_stride_blk + slot*kv_stride_tok + kvh*kv_stride_head + d
 *            (NHD = [num_blocks][block_size][Hkv][D] and HND = [num_blocks][Hkv][block_size][D]
 *             are both expressible; reading R7)
 *   block_table int32 [num_seqs][>= max_blocks_per_seq], row stride bt_stride; entries at
 *            index >= ceil(L_b / block_size) are never read (may be -1)
 *   cu_seqlens_q int32 [num_seqs + 1], cu_seqlens_q[0] == 0, nondecreasing; cu[num_seqs] == num_tokens
 *   seq_lens int32 [num_seqs]  (L_b = context + query, NOT the context length)
 *   out      [num_tokens][num_q_heads][head_dim]       strides (o_stride_tok, o_stride_head, 1)
 */
typedef struct pattn_problem {
  int32_t num_seqs;           /* B >= 1 */
  int32_t num_tokens;         /* T = sum_b q_b */
  int32_t num_q_heads;        /* Hq, multiple of num_kv_heads */
  int32_t num_kv_heads;       /* Hkv */
  int32_t head_dim;           /* D in {64, 128} */
  int32_t block_size;         /* tokens per KV block (any >= 1; 16*k uses the TMA decode path) */
  int32_t num_blocks;         /* physical blocks in each cache */
  int32_t max_blocks_per_seq; /* block-table row length */
  int32_t max_query_len;      /* hint: >= max_b q_b  (<= 0: use num_tokens) */
  int32_t max_seq_len;        /* hint: >= max_b L_b  (<= 0: use max_blocks_per_seq*block_size) */
  int32_t dtype;              /* pattn_dtype_t */
  int32_t flags;              /* PATTN_FLAG_* (0 = defaults) */
  int64_t q_stride_tok, q_stride_head;
  int64_t kv_stride_blk, kv_stride_tok, kv_stride_head;
  int64_t bt_stride;
  int64_t o_stride_tok, o_stride_head;
} pattn_problem_t;

/* flags (planner overrides, for tests and sweeps; 0 = let the planner decide) */
#define PATTN_FLAG_FORCE_GENERIC 0x1u  /* route every Q block to the generic SIMT kernel (K4) */
#define PATTN_FLAG_NO_SPLIT 0x2u       /* decode: one segment per sequence (no parallel tiled softmax) */
#define PATTN_FLAG_FORCE_SPLIT 0x4u    /* decode: always split into segments even for short sequences */
#define PATTN_FLAG_SERIAL 0x8u         /* single stream even when a second stream is supplied */
#define PATTN_FLAG_BASELINE 0x10u      /* the paper's baseline kernel (App. A): one warp per
                                          (query token, query head), tile = BLOCK_SIZE keys; for
                                          comparison only -- every row, prefill and decode */

/* Kernel kinds, for pattn_exec_opts_t.events and pattn_debug_plan(). */
enum {
  PATTN_KERNEL_METADATA = 0, /* K5: batch metadata + work lists */
  PATTN_KERNEL_PREFILL = 1,  /* K1: tcgen05/TMEM Q-block kernel */
  PATTN_KERNEL_DECODE = 2,   /* K2 / K2W: split-KV decode, "parallel tiled softmax" */
  PATTN_KERNEL_REDUCE = 3,   /* K3: segment reduction */
  PATTN_KERNEL_GENERIC = 4,  /* K4: generic SIMT Q-block kernel (fp32 path, fallback shapes) */
  PATTN_KERNEL_BASELINE = 5, /* K7: the paper's baseline kernel (PATTN_FLAG_BASELINE only) */
  PATTN_KERNEL_COUNT = 6
};

/*
 * Optional execution options (pattn_unified_attention_ex).  All fields may be
 * zero/NULL.
 *   stream2: a second stream; when given, the decode kernels run on it
 *            concurrently with the prefill kernel, joined back into `stream`
 *            with events before the call's work completes.
 *   events:  2*PATTN_KERNEL_COUNT cudaEvent_t handles (as void*); when
 *            events[2k] / events[2k+1] are non-NULL they are recorded
 *            immediately before / after the launch of kernel kind k on the
 *            stream that kernel runs on (no synchronisation).
 */
typedef struct pattn_exec_opts {
  void* stream2;
  void* events[2 * PATTN_KERNEL_COUNT];
} pattn_exec_opts_t;

/* Bytes of device workspace pattn_unified_attention needs for this problem (>= 256-byte aligned base). */
PATTN_API size_t pattn_workspace_size(const pattn_problem_t* p);

/*
 * The unified attention call (north_star: unified_attention(q, k_cache, v_cache,
 * block_table, cu_seqlens_q, seq_lens, scale, num_kv_heads, block_size, out);
 * num_kv_heads and block_size travel in *p).
 *   scale: the softmax scale (1/sqrt(head_dim) in Eq. 1; any finite value accepted).
 *   out:   written for every token row in [0, T) and every query head; nothing else
 *          in `out` is touched.
 *   workspace: device memory of >= pattn_workspace_size(p) bytes, 256-byte aligned;
 *          contents need not be initialised and are clobbered.
 * Returns PATTN_OK once the work is enqueued.
 */
PATTN_API pattn_status_t pattn_unified_attention(const pattn_problem_t* p, const void* q, const void* k_cache,
                                       const void* v_cache, const int32_t* block_table,
                                       const int32_t* cu_seqlens_q, const int32_t* seq_lens, float scale,
                                       void* out, void* workspace, size_t workspace_bytes, void* stream);

/* As pattn_unified_attention, with execution options (may be NULL). */
PATTN_API pattn_status_t pattn_unified_attention_ex(const pattn_problem_t* p, const void* q, const void* k_cache,
                                          const void* v_cache, const int32_t* block_table,
                                          const int32_t* cu_seqlens_q, const int32_t* seq_lens,
                                          float scale, void* out, void* workspace, size_t workspace_bytes,
                                          void* stream, const pattn_exec_opts_t* opts);

/*
 * End-to-end variant: q, block_table, cu_seqlens_q, seq_lens and out are HOST
 * pointers (pinned memory recommended; the table is read as [num_seqs][bt_stride]);
 * the KV caches stay device-resident (they are the server's state).  The call
 * enqueues the host->device copies, the attention and the device->host copy of
 * `out` on `stream` and returns; the caller synchronises `stream` before reading
 * out_host.  The workspace must hold pattn_hostio_workspace_size(p) bytes.
 * q_stride_* / o_stride_* describe the host arrays and must be dense
 * (q_stride_head == head_dim, q_stride_tok == Hq*head_dim; same for out).
 */
PATTN_API size_t pattn_hostio_workspace_size(const pattn_problem_t* p);
PATTN_API pattn_status_t pattn_unified_attention_hostio(const pattn_problem_t* p, const void* q_host,
                                              const void* k_cache, const void* v_cache,
                                              const int32_t* block_table_host,
                                              const int32_t* cu_seqlens_q_host, const int32_t* seq_lens_host,
                                              float scale, void* out_host, void* workspace,
                                              size_t workspace_bytes, void* stream);

/*
 * Paged KV write ("reshape and cache"): store the K and V rows of the batch's query
 * tokens into the paged caches, the step the attention call presupposes ("Q, K, and V
 * have already been computed ... and stored in the KV cache in blocks", §4.3
 * P:327, App. A; SPEC write_kv S:139-147).  For sequence b, token i in [0, q_b):
 *     pos = L_b - q_b + i ;  blk = block_table[b][pos / block_size] ;  slot = pos % block_size
 *     k_cache[blk][slot][h][:] = k_new[cu_seqlens_q[b] + i][h][:]   (h < num_kv_heads; same for V)
 * i.e. the same batch metadata as pattn_unified_attention, so a caller runs
 * pattn_write_kv then pattn_unified_attention on one stream.  A bit-exact copy.
 *   p:       uses num_seqs, num_tokens, num_kv_heads, head_dim, block_size, dtype,
 *            max_blocks_per_seq, kv_stride_*, bt_stride (the q/o fields are ignored).
 *   k_new, v_new: DEVICE [num_tokens][num_kv_heads][head_dim], strides
 *            (new_stride_tok, new_stride_head, 1) in elements, shared by both.
 *   k_cache, v_cache: DEVICE caches, written only at the addressed (blk, slot) rows.
 * Every row start must be 16-byte aligned (else PATTN_ERR_UNSUPPORTED).  Metadata is
 * trusted as in pattn_unified_attention (validate with pattn_validate_metadata_host);
 * two tokens addressing the same (blk, slot) is a caller error (last writer undefined).
 * num_tokens == 0 is a no-op.  Asynchronous on `stream`.
 */
PATTN_API pattn_status_t pattn_write_kv(const pattn_problem_t* p, const void* k_new, const void* v_new,
                                        int64_t new_stride_tok, int64_t new_stride_head, void* k_cache,
                                        void* v_cache, const int32_t* block_table, const int32_t* cu_seqlens_q,
                                        const int32_t* seq_lens, void* stream);

/*
 * Tuning heuristics (the paper's two-step flow, §4.2: micro-benchmark sweeps
 * outside the runtime, results "export[ed] as heuristics --- simple if-else decision
 * trees" that also cover scenarios not in the sweep).  A tree maps host-known batch
 * features to the planner's launch knobs (H1); libpattn consults it in every call.
 * Precedence: PATTN_* environment overrides > the loaded tree > built-in defaults.
 */
typedef struct pattn_tuning {
  int32_t items_per_sm;       /* decode: target work items per SM -- K2: (segment x KV head x head group),
                                 K2W: (segment x group of HB KV heads) -- (default 16 for K2, 2 for K2W) */
  int32_t min_chunk_tokens;   /* decode: shortest split segment, in keys (default 256 for K2, 128 for K2W) */
  int32_t decode_ctas_per_sm; /* decode: resident K2 CTAs per SM, 1..4 (default 2; K2W runs one) */
  int32_t k2_sm_mbs;          /* mixed batches, two streams: decode streaming rate per SM (MB/s) that K5's
                                 SM-partition model assumes -- higher leaves more SMs to the prefill kernel
                                 (default: the measured rate of the decode kernel in use, K2W 100000, K2 61000) */
  int32_t serial;             /* mixed batches: 1 = prefill and decode kernels back to back on one stream
                                 even when a second stream is given; 0 = concurrent (default) */
  int32_t decode_kernel;      /* decode kernel: 1 = K2W (head-wide TMA boxes) where it applies (G <= 16,
                                 2 | Hkv), 2 = K2 (one KV head per work item); default 1 */
} pattn_tuning_t;           /* 0 in a field = built-in default */

enum {
  PATTN_FEAT_NUM_SEQS = 0,      /* num_seqs */
  PATTN_FEAT_NUM_TOKENS = 1,    /* num_tokens */
  PATTN_FEAT_MAX_QUERY_LEN = 2, /* max_query_len hint (<= 0: num_tokens) -- 1 means a decode-only batch */
  PATTN_FEAT_MAX_SEQ_LEN = 3,   /* max_seq_len hint (<= 0: max_blocks_per_seq * block_size) */
  PATTN_FEAT_COUNT = 4
};

/* One node of a decision tree, stored as an array with the root at index 0.
 * Internal node: feature in [0, PATTN_FEAT_COUNT), children lt / ge with index > this
 * node's (so every tree is finite and acyclic): value < threshold -> lt, else ge.
 * Leaf: feature = -1; `leaf` holds the knobs. */
typedef struct pattn_tree_node {
  int32_t feature;
  int32_t lt, ge;
  double threshold;
  pattn_tuning_t leaf;
} pattn_tree_node_t;

/* Install (copy) a tree for all later calls in this process; nodes == NULL or n_nodes == 0
 * removes it.  A malformed tree (bad feature, child index <= parent or >= n_nodes, leaf
 * knobs out of range) returns PATTN_ERR_INVALID_ARG and leaves the current tree in place.
 * Thread-safe; not meant to be called concurrently with in-flight planning of other threads. */
PATTN_API pattn_status_t pattn_set_tuning_tree(const pattn_tree_node_t* nodes, int32_t n_nodes);

/* Host-only: the knobs the planner will use for problem p (tree leaf, env overrides and
 * defaults resolved), written to *out.  No device work. */
PATTN_API pattn_status_t pattn_plan_tuning(const pattn_problem_t* p, pattn_tuning_t* out);

/*
 * CUDA-graph capture of the unified call ("full graph" execution, §6.2 P:180-199:
 * graphs are recorded per batch-size bucket at startup and replayed; the static launch grid
 * of §4.7 P:401-406 makes one recording valid for every batch that fits the bucket).
 *   pattn_graph_capture: records ONE pattn_unified_attention_ex call on `stream` (with
 *     `stream2` as the concurrent decode branch when non-NULL) into an executable graph.
 *     Every pointer passed is baked into the graph: they must stay valid, and the caller
 *     refreshes the CONTENTS of q / block_table / cu_seqlens_q / seq_lens between launches
 *     (the grids never depend on them; sequences with q_b = 0 pad a bucket).  Sizes in *p
 *     (num_seqs, num_tokens, hints) are the bucket's capacities.  `stream` must not be
 *     capturing already.  Returns PATTN_OK and a handle in *graph.
 *   pattn_graph_launch: replays the graph on `stream` (asynchronous).
 *   pattn_graph_destroy: frees the handle (host-side graph objects only; no device memory
 *     is owned).  The graph must not be in flight.
 */
typedef struct pattn_graph* pattn_graph_t;
PATTN_API pattn_status_t pattn_graph_capture(const pattn_problem_t* p, const void* q, const void* k_cache,
                                             const void* v_cache, const int32_t* block_table,
                                             const int32_t* cu_seqlens_q, const int32_t* seq_lens, float scale,
                                             void* out, void* workspace, size_t workspace_bytes, void* stream,
                                             void* stream2, pattn_graph_t* graph);
PATTN_API pattn_status_t pattn_graph_launch(pattn_graph_t graph, void* stream);
PATTN_API pattn_status_t pattn_graph_destroy(pattn_graph_t graph);

/* Static string for a status code. */
PATTN_API const char* pattn_status_string(pattn_status_t s);

/*
 * Host-side validation of HOST copies of the metadata (SPEC error taxonomy):
 * cu_seqlens_q[0] == 0, 0 <= q_b <= L_b, cu[B] == num_tokens -> INVALID_SEQUENCE;
 * ceil(L_b/bs) > max_blocks_per_seq or a used block id outside [0, num_blocks)
 * -> INDEX_OUT_OF_RANGE; num_seqs == 0 -> EMPTY_BATCH.  No device work.
 */
PATTN_API pattn_status_t pattn_validate_metadata_host(const pattn_problem_t* p, const int32_t* cu_seqlens_q_host,
                                            const int32_t* seq_lens_host, const int32_t* block_table_host);

/*
 * Test/introspection: run only the metadata kernel (K5) for this problem and copy
 * its results into the caller's DEVICE buffer `plan_out` (int32, plan_capacity
 * entries) with cudaMemcpyAsync on `stream`.  Layout:
 *   [0] total prefill Q blocks   [1] number of decode sequences   [2] decode chunks (segments)
 *   [3] BLOCK_Q used for prefill [4] decode chunk size in KV blocks
 *   [8 .. 8+B]      cu_q_blocks (prefill Q blocks per sequence, exclusive scan; decodes count 0)
 *   [8+B+1 .. 8+2B+1] cu_chunks (decode segments per sequence, exclusive scan; non-decodes count 0)
 * plan_capacity must be >= 2*num_seqs + 10.
 */
PATTN_API pattn_status_t pattn_debug_plan(const pattn_problem_t* p, const int32_t* cu_seqlens_q, const int32_t* seq_lens,
                                int32_t* plan_out, int32_t plan_capacity, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Number of kernel launches pattn_unified_attention enqueues for this problem (host-side plan). */
PATTN_API int32_t pattn_planned_launches(const pattn_problem_t* p);

/* Bit mask of the kernel kinds (1 << PATTN_KERNEL_*) pattn_unified_attention launches for this problem,
 * plus PATTN_PLAN_DECODE_WIDE when the decode kind runs as K2W (head-wide TMA boxes, HB KV heads per
 * work item; k2w_decode.cu) rather than K2. */
#define PATTN_PLAN_DECODE_WIDE (1 << 8)
PATTN_API int32_t pattn_planned_kernels(const pattn_problem_t* p);

/* Text of the CUDA error behind the calling thread's last PATTN_ERR_CUDA ("" if none). */
PATTN_API const char* pattn_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
PATTN_API int32_t pattn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PATTN_H_ */
