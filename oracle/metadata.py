"""Batch metadata and index arithmetic of the paper's kernels, written out plainly.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* build_batch_meta: query/context lengths, Q blocks per sequence
  = ceil(query_length / BLOCK_Q), one per decode, the accumulated
  Q-block tensor and the decode count (a decode is q_b == 1,
  reading R15).
* seq_index_lookup: the sequence owning a global (token or Q-block) index --
  the last i with cu[i] <= idx (App. A, App. B; ties from empty
  sequences resolved as in reading R14).  Linear scan, not a binary search.
* kv_head_for_query_head: h // (Hq / Hkv) (App. A, reading R3).
* qblock_rows: the (token, head) pairs of a Q block, token-major head-minor
  (reading R8).
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np


def build_batch_meta(cu_seqlens_q, seq_lens, block_q: int) -> Dict[str, np.ndarray]:
    cu = [int(x) for x in cu_seqlens_q]
    sl = [int(x) for x in seq_lens]
    B = len(sl)
    q_lens, ctx_lens, nqb, is_decode = [], [], [], []
    for b in range(B):
        q = cu[b + 1] - cu[b]
        if q < 0 or q > sl[b]:
            raise ValueError("InvalidSequence")
        q_lens.append(q)
        ctx_lens.append(sl[b] - q)
        nqb.append((q + block_q - 1) // block_q)
        is_decode.append(q == 1)
    cu_qb = [0]
    for n in nqb:
        cu_qb.append(cu_qb[-1] + n)
    return dict(
        q_lens=np.array(q_lens, np.int64),
        ctx_lens=np.array(ctx_lens, np.int64),
        num_q_blocks=np.array(nqb, np.int64),
        cu_q_blocks=np.array(cu_qb, np.int64),
        is_decode=np.array(is_decode, bool),
        num_decodes=int(sum(is_decode)),
        total_q_blocks=cu_qb[-1],
    )


def seq_index_lookup(cu, idx: int) -> int:
    cu = [int(x) for x in cu]
    if not (0 <= idx < cu[-1]):
        raise IndexError("IndexOutOfRange")
    best = -1
    for i in range(len(cu) - 1):
        if cu[i] <= idx:
            best = i
    return best


def kv_head_for_query_head(h: int, num_q_heads: int, num_kv_heads: int) -> int:
    if not (0 <= h < num_q_heads):
        raise IndexError("IndexOutOfRange")
    return h // (num_q_heads // num_kv_heads)


def qblock_rows(q_block_in_seq: int, block_q: int, q_len: int, kv_head: int, G: int) -> List[Tuple[int, int]]:
    """Valid (token-in-seq, q_head) rows of a Q block; rows past q_len are padding (not listed)."""
    rows = []
    for r in range(block_q * G):
        tok = q_block_in_seq * block_q + r // G
        if tok < q_len:
            rows.append((tok, kv_head * G + r % G))
    return rows


def paged_slot(block_table_row, t: int, block_size: int) -> Tuple[int, int]:
    """Key position t -> (physical block, slot)."""
    return int(block_table_row[t // block_size]), t % block_size
