"""Pure-Python brute-force paged attention for tiny inputs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

An independent second implementation of the definition in pattn_oracle.c,
written without numpy arithmetic: Python floats (IEEE fp64), math.exp and
math.fsum (exactly rounded sums).  Used only to pin oracle.attention on small
batches (<= a few thousand (row, key) pairs).

Follows: Eq. 1 and Eq. 2; terminology:
a query row at index i of a sequence with context ctx sees keys 0..ctx+i.
"""
from __future__ import annotations

import math
from typing import List


def _f(x) -> float:
    return float(x)


def attention(q, k_rows_of, v_rows_of, cu_seqlens_q, seq_lens, scale, num_q_heads, num_kv_heads):
    """q: nested [T][Hq][D] floats; k_rows_of(b, t, g) / v_rows_of(b, t, g) -> list of D floats
    for key position t of sequence b, KV head g (the caller resolves the block table).
    Returns nested [T][Hq][D] floats."""
    G = num_q_heads // num_kv_heads
    B = len(seq_lens)
    T = cu_seqlens_q[B]
    out: List = [None] * T
    for b in range(B):
        qb = cu_seqlens_q[b + 1] - cu_seqlens_q[b]
        ctx = seq_lens[b] - qb
        for i in range(qb):
            tok = cu_seqlens_q[b] + i
            row = []
            for h in range(num_q_heads):
                g = h // G
                n = ctx + i + 1
                qv = [_f(x) for x in q[tok][h]]
                s = []
                for t in range(n):
                    kv = k_rows_of(b, t, g)
                    s.append(_f(scale) * math.fsum(a * _f(c) for a, c in zip(qv, kv)))
                m = max(s)
                w = [math.exp(x - m) for x in s]
                den = math.fsum(w)
                D = len(qv)
                vs = [v_rows_of(b, t, g) for t in range(n)]
                row.append([math.fsum(w[t] * _f(vs[t][d]) for t in range(n)) / den for d in range(D)])
            out[tok] = row
    return out


def batch_attention(batch):
    """Run on a workloads.Batch (NHD or HND), resolving pages with plain indexing."""
    from .attention import widen  # storage widening only (bf16 bits -> fp32)

    w = batch.workload
    q = widen(batch.q).tolist()
    kc = widen(batch.k_cache)
    vc = widen(batch.v_cache)
    bt = batch.block_table.tolist()
    bs = w.block_size

    def rows(cache):
        def get(b, t, g):
            blk = bt[b][t // bs]
            if batch.layout == "NHD":
                return cache[blk, t % bs, g, :].tolist()
            return cache[blk, g, t % bs, :].tolist()

        return get

    return attention(q, rows(kc), rows(vc), batch.cu_seqlens_q.tolist(), batch.seq_lens.tolist(), w.scale,
                     w.num_q_heads, w.num_kv_heads)
