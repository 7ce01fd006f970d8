"""Paged KV write oracle ("reshape and cache").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it computes: the cache state the attention call presupposes -- "Q, K, and V have
already been computed before the kernel launch and stored in the KV cache in blocks"
(§4.3; App. A) -- written through the block table with SPEC's
write_kv addressing: logical position t of sequence b lives in physical block
block_table[b][t // BLOCK_SIZE] at slot t % BLOCK_SIZE.  The batch's query
tokens are the newest tokens of each sequence: token i of sequence b has position
ctx_b + i, ctx_b = L_b - q_b (terminology, §4.2).

Pure-Python loops over (sequence, token); arrays are copied element-for-element (no
arithmetic), so the result is exact in any dtype.
Pins (tests/test_oracle_kvcache.py): SPEC's worked example (pos 17, bs 16 -> table[1],
slot 1), the identity block table reducing to a plain reshape, injectivity /
untouched-slot checks, and round trip through the attention oracle (constant-V).
"""
from __future__ import annotations

import numpy as np


def write_kv(k_new, v_new, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, block_size):
    """Return (k_cache', v_cache'): copies of the caches with the batch's K/V rows stored.

    k_new, v_new: [T, Hkv, D]; caches: [num_blocks, block_size, Hkv, D] (any dtype, incl.
    bf16 bit patterns as uint16); block_table [B, max_blocks]; cu_seqlens_q [B+1];
    seq_lens [B] (L_b = context + query).
    """
    kc = np.array(k_cache, copy=True)
    vc = np.array(v_cache, copy=True)
    cu = [int(x) for x in cu_seqlens_q]
    for b in range(len(seq_lens)):
        q_b = cu[b + 1] - cu[b]
        ctx_b = int(seq_lens[b]) - q_b
        for i in range(q_b):
            pos = ctx_b + i
            blk = int(block_table[b][pos // block_size])
            slot = pos % block_size
            kc[blk, slot, :, :] = k_new[cu[b] + i]
            vc[blk, slot, :, :] = v_new[cu[b] + i]
    return kc, vc
