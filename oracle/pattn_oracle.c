/*
 * oracle/pattn_oracle.c -- fp64 CPU oracle of unified paged causal attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2511_11581_b200/csrc) and
 * includes nothing from it.
 *
 * What it computes (the plain definition, no tiling, no online softmax):
 *
 *   for every sequence b:                       (Terminology, §4.2)
 *     q_b   = cu_seqlens_q[b+1] - cu_seqlens_q[b]      query length
 *     L_b   = seq_lens[b]                              sequence length = context + query
 *     ctx_b = L_b - q_b                                context length
 *     for every query row i in [0, q_b) and query head h:
 *       g = h / (Hq / Hkv)                     GQA: contiguous groups share a KV head (reading R3)
 *       n = ctx_b + i + 1                      keys 0 .. ctx_b+i, self-inclusive (reading R1/R2)
 *       for t in [0, n):                       K/V of all tokens are in the paged cache
 *         blk = block_table[b][t / bs], slot = t % bs
 *         s_t = scale * sum_d q[tok][h][d] * K[blk][slot][g][d]      Eq. 1
 *       M = max_t s_t ; w_t = exp(s_t - M)                            Eq. 2
 *       out[tok][h][:] = sum_t w_t V[blk_t][slot_t][g][:] / sum_t w_t
 *
 * Inputs are the exact values the GPU sees (fp32, or bf16 already widened to
 * fp32 exactly); every product and sum is fp64.  Threaded over output rows with
 * OpenMP; each row is independent so the thread count does not change results.
 *
 * Parity pins: tests/test_oracle_pins.py (dense SDPA special case, pure-Python
 * brute force, closed forms, invariants).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_ARG 1
#define ORACLE_ERR_SEQUENCE 3 /* q_b < 0 or q_b > L_b (InvalidSequence) */
#define ORACLE_ERR_INDEX 4    /* block id out of range (IndexOutOfRange) */

/* Sequence owning query token `tok`: the b with cu[b] <= tok < cu[b+1] (App. A). */
static int seq_of_token(const int32_t* cu, int num_seqs, int64_t tok) {
  for (int b = 0; b < num_seqs; ++b)
    if (cu[b] <= tok && tok < cu[b + 1]) return b;
  return -1;
}

int oracle_validate(int num_seqs, const int32_t* cu, const int32_t* seq_lens, int block_size,
                    int num_blocks, const int32_t* block_table, int64_t bt_stride, int max_blocks_per_seq) {
  if (num_seqs < 0 || block_size <= 0) return ORACLE_ERR_ARG;
  if (cu[0] != 0) return ORACLE_ERR_SEQUENCE;
  for (int b = 0; b < num_seqs; ++b) {
    int64_t qb = (int64_t)cu[b + 1] - cu[b];
    if (qb < 0 || qb > seq_lens[b]) return ORACLE_ERR_SEQUENCE;
    int64_t nblk = ((int64_t)seq_lens[b] + block_size - 1) / block_size;
    if (nblk > max_blocks_per_seq) return ORACLE_ERR_INDEX;
    for (int64_t j = 0; j < nblk; ++j) {
      int32_t id = block_table[(int64_t)b * bt_stride + j];
      if (id < 0 || id >= num_blocks) return ORACLE_ERR_INDEX;
    }
  }
  return ORACLE_OK;
}

/*
 * rows: optional list of output rows, row = tok * Hq + h (NULL => all T*Hq rows in order).
 * out:  fp64, [n_rows][head_dim] (row-major, contiguous).
 */
int oracle_paged_attention(int num_seqs, const int32_t* cu_seqlens_q, const int32_t* seq_lens,
                           int num_q_heads, int num_kv_heads, int head_dim, int block_size,
                           const float* q, int64_t q_stride_tok, int64_t q_stride_head,
                           const float* k_cache, const float* v_cache, int64_t kv_stride_blk,
                           int64_t kv_stride_tok, int64_t kv_stride_head, const int32_t* block_table,
                           int64_t bt_stride, double scale, const int64_t* rows, int64_t n_rows,
                           double* out, int num_threads) {
  if (num_q_heads <= 0 || num_kv_heads <= 0 || num_q_heads % num_kv_heads != 0 || head_dim <= 0)
    return ORACLE_ERR_ARG;
  const int G = num_q_heads / num_kv_heads;
  const int64_t T = cu_seqlens_q[num_seqs];
  if (rows == NULL) n_rows = T * num_q_heads;
#ifdef _OPENMP
  if (num_threads > 0) omp_set_num_threads(num_threads);
#endif
  int err = ORACLE_OK;

#pragma omp parallel
  {
    int64_t cap = 0;
    double* s = NULL;
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < n_rows; ++r) {
      int64_t row = rows ? rows[r] : r;
      int64_t tok = row / num_q_heads;
      int h = (int)(row % num_q_heads);
      double* o = out + r * head_dim;
      int b = seq_of_token(cu_seqlens_q, num_seqs, tok);
      if (b < 0 || tok >= T) {
#pragma omp atomic write
        err = ORACLE_ERR_ARG;
        continue;
      }
      int64_t qb = (int64_t)cu_seqlens_q[b + 1] - cu_seqlens_q[b];
      int64_t ctx = (int64_t)seq_lens[b] - qb;
      int64_t i = tok - cu_seqlens_q[b];
      int64_t n = ctx + i + 1;
      int g = h / G;
      if (n > cap) {
        free(s);
        cap = n;
        s = (double*)malloc(sizeof(double) * (size_t)cap);
      }
      const float* qv = q + tok * q_stride_tok + (int64_t)h * q_stride_head;
      double M = -INFINITY;
      for (int64_t t = 0; t < n; ++t) {
        int32_t blk = block_table[(int64_t)b * bt_stride + t / block_size];
        const float* kv = k_cache + (int64_t)blk * kv_stride_blk + (t % block_size) * kv_stride_tok +
                          (int64_t)g * kv_stride_head;
        double dot = 0.0;
        for (int d = 0; d < head_dim; ++d) dot += (double)qv[d] * (double)kv[d];
        s[t] = scale * dot;
        if (s[t] > M) M = s[t];
      }
      double den = 0.0;
      for (int d = 0; d < head_dim; ++d) o[d] = 0.0;
      for (int64_t t = 0; t < n; ++t) {
        double w = exp(s[t] - M);
        den += w;
        int32_t blk = block_table[(int64_t)b * bt_stride + t / block_size];
        const float* vv = v_cache + (int64_t)blk * kv_stride_blk + (t % block_size) * kv_stride_tok +
                          (int64_t)g * kv_stride_head;
        for (int d = 0; d < head_dim; ++d) o[d] += w * (double)vv[d];
      }
      for (int d = 0; d < head_dim; ++d) o[d] /= den;
    }
    free(s);
  }
  return err;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
