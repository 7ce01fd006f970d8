"""Pins for the fp64 paged-attention oracle (oracle/pattn_oracle.c) against things
other than itself: a pure-Python brute force (independent implementation), the
dense library routine torch SDPA in float64 (special case: K/V gathered out of
the pages, explicit bottom-right causal mask), closed forms (constant V, single
key, uniform scores, needle) and invariants (causality, physical-block
permutation, cache layout).  A dropped term, a wrong sign, an off-by-one in the
causal extent, a transposed GQA map or a wrong page lookup fails at least one.
"""
import math

import numpy as np
import pytest
import torch

from oracle import attention as O
from oracle import brute
from workloads import CONFIGS, Workload, generate
from workloads.gen import random_workload

TOL = 1e-12


def _gather_dense(batch, b, cache):
    """K or V rows 0..L_b-1 of sequence b, shape [L_b, Hkv, D] (test-side page walk)."""
    w = batch.workload
    L = int(batch.seq_lens[b])
    c = O.widen(cache).astype(np.float64)
    rows = []
    for t in range(L):
        blk = batch.block_table[b, t // w.block_size]
        if batch.layout == "NHD":
            rows.append(c[blk, t % w.block_size])
        else:
            rows.append(c[blk, :, t % w.block_size])
    return np.stack(rows)


def _sdpa_reference(batch):
    """torch scaled_dot_product_attention, float64, per sequence, enable_gqa, explicit mask
    (query i of a sequence with context ctx sees keys t <= ctx + i; NOT is_causal, which is
    top-left aligned)."""
    w = batch.workload
    q = O.widen(batch.q).astype(np.float64)
    out = np.zeros_like(q)
    for b in range(w.num_seqs):
        s, e = int(batch.cu_seqlens_q[b]), int(batch.cu_seqlens_q[b + 1])
        if e == s:
            continue
        L = int(batch.seq_lens[b])
        ctx = L - (e - s)
        K = torch.from_numpy(_gather_dense(batch, b, batch.k_cache)).permute(1, 0, 2)[None]
        V = torch.from_numpy(_gather_dense(batch, b, batch.v_cache)).permute(1, 0, 2)[None]
        Q = torch.from_numpy(q[s:e]).permute(1, 0, 2)[None]
        i = torch.arange(e - s)[:, None]
        t = torch.arange(L)[None, :]
        mask = t <= ctx + i
        o = torch.nn.functional.scaled_dot_product_attention(
            Q, K, V, attn_mask=mask, scale=w.scale, enable_gqa=True
        )
        out[s:e] = o[0].permute(1, 0, 2).numpy()
    return out


def test_config1_vs_bruteforce():
    batch = generate(CONFIGS["c1_tiny"], seed=1001)
    ref = O.batch_attention(batch)
    bf = np.array(brute.batch_attention(batch))
    assert np.isfinite(ref).all()
    np.testing.assert_allclose(ref, bf, rtol=0, atol=TOL)


@pytest.mark.parametrize("seed", range(6))
def test_random_tiny_vs_bruteforce(seed):
    rng = np.random.default_rng(seed)
    heads = [(4, 1), (4, 2), (2, 2), (6, 3)][seed % 4]
    bs = [16, 5, 8, 3][seed % 4]
    w = random_workload(rng, heads, head_dim=8, block_size=bs, dtype=["f32", "bf16"][seed % 2],
                        max_seqs=3, max_len=24)
    batch = generate(w, seed=seed, layout=["NHD", "HND"][seed % 2])
    ref = O.batch_attention(batch)
    bf = np.array(brute.batch_attention(batch))
    np.testing.assert_allclose(ref, bf, rtol=0, atol=TOL)


@pytest.mark.parametrize("seed", range(5))
def test_random_vs_sdpa_fp64(seed):
    rng = np.random.default_rng(100 + seed)
    heads = [(32, 8), (8, 8), (16, 1), (4, 2), (64, 8)][seed]
    w = random_workload(rng, heads, head_dim=[64, 128][seed % 2], block_size=[16, 80, 16, 7, 32][seed],
                        dtype=["bf16", "f32"][seed % 2], max_seqs=5, max_len=200)
    batch = generate(w, seed=seed, dist=["uniform", "peaked"][seed % 2], layout=["NHD", "HND"][seed % 2])
    np.testing.assert_allclose(O.batch_attention(batch), _sdpa_reference(batch), rtol=0, atol=1e-11)


def test_constant_v_gives_v():
    w = Workload("cv", ((0, 9), (20, 1), (7, 5)), 8, 2, 16, 4, "f32")
    batch = generate(w, seed=3, poison=False)
    vec = np.random.default_rng(0).uniform(-1, 1, size=(2, 16)).astype(np.float32)
    batch.v_cache[:] = vec[None, None, :, :]
    out = O.batch_attention(batch)
    exp = np.repeat(vec, 4, axis=0)  # q head h -> kv head h // 4
    np.testing.assert_allclose(out, np.broadcast_to(exp, out.shape), rtol=0, atol=1e-14)


def test_single_key_and_first_prefill_row():
    # (ctx 0, q 1): one visible key -> the output is exactly that key's V row
    # prefill (ctx 0, q 6): row 0 sees only itself (self-inclusive reading R1)
    w = Workload("one", ((0, 1), (0, 6)), 4, 2, 8, 4, "bf16")
    batch = generate(w, seed=4)
    out = O.batch_attention(batch)
    v = O.widen(batch.v_cache)
    for b, tok in ((0, 0), (1, 1)):
        blk = batch.block_table[b, 0]
        for h in range(4):
            np.testing.assert_array_equal(out[tok, h], v[blk, 0, h // 2].astype(np.float64))


def test_uniform_scores_give_mean_of_visible_v():
    w = Workload("zq", ((0, 7), (13, 3), (30, 1)), 4, 1, 8, 4, "f32")
    batch = generate(w, seed=5, dist="zero_q")
    out = O.batch_attention(batch)
    for b in range(w.num_seqs):
        V = _gather_dense(batch, b, batch.v_cache)
        s = int(batch.cu_seqlens_q[b])
        q = int(batch.cu_seqlens_q[b + 1]) - s
        ctx = int(batch.seq_lens[b]) - q
        for i in range(q):
            mean = V[: ctx + i + 1, 0].mean(axis=0)
            for h in range(4):
                np.testing.assert_allclose(out[s + i, h], mean, rtol=0, atol=1e-14)


def test_needle_selects_its_value_row():
    w = Workload("nd", ((40, 1), (0, 12), (70, 3)), 8, 2, 128, 16, "bf16")
    batch = generate(w, seed=6, dist="needle")
    out = O.batch_attention(batch)
    v = O.widen(batch.v_cache)
    for b in range(w.num_seqs):
        s, e = int(batch.cu_seqlens_q[b]), int(batch.cu_seqlens_q[b + 1])
        for g in range(2):
            t = int(batch.needle_pos[b, g])
            row = v[batch.block_table[b, t // 16], t % 16, g].astype(np.float64)
            for h in range(g * 4, g * 4 + 4):
                np.testing.assert_allclose(out[s:e, h], np.broadcast_to(row, (e - s, 128)), rtol=0, atol=1e-14)


def test_causality_point_perturbation():
    w = Workload("ca", ((10, 6), (0, 9)), 4, 2, 16, 4, "f32")
    batch = generate(w, seed=7)
    base = O.batch_attention(batch)
    for b, p in ((0, 12), (1, 4)):
        pert = generate(w, seed=7)
        blk = pert.block_table[b, p // 4]
        pert.k_cache[blk, p % 4] += 0.5
        pert.v_cache[blk, p % 4] -= 0.25
        out = O.batch_attention(pert)
        s, e = int(batch.cu_seqlens_q[b]), int(batch.cu_seqlens_q[b + 1])
        ctx = int(batch.seq_lens[b]) - (e - s)
        for i in range(e - s):
            if ctx + i < p:
                np.testing.assert_array_equal(out[s + i], base[s + i])
            else:
                assert np.abs(out[s + i] - base[s + i]).max() > 1e-6
        other = [x for x in range(w.num_tokens) if not (s <= x < e)]
        np.testing.assert_array_equal(out[other], base[other])


def test_physical_block_permutation_and_layout_invariance():
    w = Workload("perm", ((33, 1), (0, 20), (5, 17)), 8, 2, 32, 8, "bf16")
    a = generate(w, seed=8, permute_blocks=False, poison=True)
    b = generate(w, seed=8, permute_blocks=False, poison=True)
    # move every block to a new physical slot and rewrite the table (data follows the pages)
    perm = np.random.default_rng(1).permutation(a.num_blocks)
    b.k_cache = np.empty_like(a.k_cache)
    b.v_cache = np.empty_like(a.v_cache)
    b.k_cache[perm] = a.k_cache
    b.v_cache[perm] = a.v_cache
    b.block_table = np.where(a.block_table >= 0, perm[np.maximum(a.block_table, 0)], -1).astype(np.int32)
    ra = O.batch_attention(a)
    np.testing.assert_array_equal(ra, O.batch_attention(b))
    h = generate(w, seed=8, permute_blocks=False, poison=True, layout="HND")
    np.testing.assert_array_equal(ra, O.batch_attention(h))


def test_scale_zero_is_uniform_average():
    w = Workload("s0", ((6, 4),), 2, 1, 8, 4, "f32")
    batch = generate(w, seed=9)
    out = O.paged_attention(batch.q, batch.k_cache, batch.v_cache, batch.block_table, batch.cu_seqlens_q,
                            batch.seq_lens, 0.0, 1, 4)
    V = _gather_dense(batch, 0, batch.v_cache)
    for i in range(4):
        np.testing.assert_allclose(out[i, 0], V[: 6 + i + 1, 0].mean(axis=0), rtol=0, atol=1e-14)


def test_overflow_bait_is_finite():
    w = Workload("big", ((50, 3),), 4, 1, 64, 16, "f32")
    batch = generate(w, seed=10, poison=False)
    batch.q *= 3000.0  # |scores| ~ 1e4
    out = O.batch_attention(batch)
    assert np.isfinite(out).all()
    assert np.abs(out).max() <= 1.0 + 1e-12  # a convex combination of V rows in [-1, 1]


def test_rows_subset_matches_full():
    w = CONFIGS["c1_tiny"]
    batch = generate(w, seed=11)
    full = O.batch_attention(batch).reshape(-1, w.head_dim)
    rows = [0, 5, 17, 33, 67]
    np.testing.assert_array_equal(O.batch_attention(batch, rows=rows), full[rows])


def test_validate_codes():
    cu = np.array([0, 3, 4], np.int32)
    sl = np.array([3, 5], np.int32)
    bt = np.array([[0, -1], [1, 2]], np.int32)
    assert O.validate(cu, sl, 4, 3, bt) == 0
    assert O.validate(cu, np.array([2, 5], np.int32), 4, 3, bt) == 3  # q_b > L_b
    assert O.validate(cu, sl, 4, 2, bt) == 4  # block id 2 >= num_blocks


def test_widen_matches_torch_bf16_to_fp32():
    """oracle.attention.widen (bf16 bit pattern -> fp32) pinned to torch's own bf16 -> fp32
    conversion on every one of the 65536 bit patterns (NaN payloads compared as NaN), and to
    closed-form values: 0x3F80 = 1.0, 0xC000 = -2.0, 0x7F80 = +inf, 0x0001 = 2^-133."""
    import torch

    from oracle.attention import widen

    bits = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    ours = widen(bits)
    ref = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float().numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    w = widen(np.array([0x3F80, 0xC000, 0x7F80, 0x0001], np.uint16))
    assert w[0] == 1.0 and w[1] == -2.0 and np.isinf(w[2]) and w[2] > 0 and w[3] == np.float32(2.0 ** -133)
    f = np.array([0.5, -3.25], np.float32)
    assert np.array_equal(widen(f), f)  # fp32 storage passes through unchanged
    # fp16 storage (PATTN_DTYPE_F16): every pattern widened exactly, as torch converts it
    h = bits.view(np.float16)
    ours16 = widen(h)
    ref16 = torch.from_numpy(h.copy()).float().numpy()
    nan16 = np.isnan(ref16)
    assert np.array_equal(np.isnan(ours16), nan16)
    assert np.array_equal(ours16[~nan16].view(np.uint32), ref16[~nan16].view(np.uint32))
    assert widen(np.array([1.0, 65504.0, 2.0 ** -24], np.float16)).tolist() == [1.0, 65504.0, 2.0 ** -24]
