"""Pins of oracle/kvcache.py (the paged KV write, §4.3, App. A P:10-14;
SPEC write_kv S:139-147) against things other than itself."""
import numpy as np

from oracle import attention as O
from oracle import kvcache as KV
from workloads import Workload, generate


def _nan_cache(nb, bs, hkv, d):
    return np.full((nb, bs, hkv, d), np.nan, np.float32)


def test_spec_worked_example_pos17_bs16():
    # "write then read at (pos=17, block_size=16) hits block table[1], slot 1"
    kc, vc = _nan_cache(8, 16, 1, 4), _nan_cache(8, 16, 1, 4)
    bt = np.array([[5, 2]], np.int32)
    k = np.array([[[1.0, 2.0, 3.0, 4.0]]], np.float32)
    v = -k
    # one sequence whose single query token sits at position 17: ctx 17, q 1, L 18
    k2, v2 = KV.write_kv(k, v, kc, vc, bt, np.array([0, 1], np.int32), np.array([18], np.int32), 16)
    assert (k2[2, 1, 0] == k[0, 0]).all() and (v2[2, 1, 0] == v[0, 0]).all()
    assert np.isnan(np.delete(k2.reshape(-1, 4), 2 * 16 + 1, axis=0)).all()  # nothing else written


def test_spec_zero_vector_roundtrip():
    # write k = 0-vector -> read returns the 0-vector
    kc, vc = _nan_cache(2, 4, 2, 8), _nan_cache(2, 4, 2, 8)
    z = np.zeros((1, 2, 8), np.float32)
    k2, _ = KV.write_kv(z, z, kc, vc, np.array([[1, 0]], np.int32), np.array([0, 1], np.int32),
                        np.array([6], np.int32), 4)
    assert (k2[0, 1] == 0).all()


def test_identity_table_is_a_reshape():
    # with block_table[b][j] = b*nb + j the paged cache of sequence b is the contiguous
    # [nb*bs] token range reshaped, so the write must equal a slice assignment
    rng = np.random.default_rng(5)
    bs, hkv, d, nb = 16, 2, 8, 4
    seqs = [(0, 40), (17, 1), (30, 20), (63, 1)]  # (ctx, q)
    B = len(seqs)
    bt = np.arange(B * nb, dtype=np.int32).reshape(B, nb)
    T = sum(q for _, q in seqs)
    k = rng.standard_normal((T, hkv, d)).astype(np.float32)
    v = rng.standard_normal((T, hkv, d)).astype(np.float32)
    cu = np.concatenate([[0], np.cumsum([q for _, q in seqs])]).astype(np.int32)
    sl = np.array([c + q for c, q in seqs], np.int32)
    kc, vc = KV.write_kv(k, v, _nan_cache(B * nb, bs, hkv, d), _nan_cache(B * nb, bs, hkv, d), bt, cu, sl, bs)
    dense_k = kc.reshape(B, nb * bs, hkv, d)
    dense_v = vc.reshape(B, nb * bs, hkv, d)
    for b, (c, q) in enumerate(seqs):
        assert (dense_k[b, c:c + q] == k[cu[b]:cu[b + 1]]).all()
        assert (dense_v[b, c:c + q] == v[cu[b]:cu[b + 1]]).all()
        assert np.isnan(dense_k[b, :c]).all() and np.isnan(dense_k[b, c + q:]).all()


def test_injective_on_permuted_table():
    # distinct (pos, kv_head) never alias: exactly T*Hkv rows change
    w = Workload("kvw", ((0, 37), (100, 1), (5, 12), (0, 1)), 8, 4, 16, 16, "f32")
    b = generate(w, seed=9)
    rng = np.random.default_rng(3)
    T = w.num_tokens
    k = rng.standard_normal((T, 4, 16)).astype(np.float32)
    kc0 = np.full_like(b.k_cache, np.nan)
    kc, _ = KV.write_kv(k, k, kc0, kc0, b.block_table, b.cu_seqlens_q, b.seq_lens, 16)
    written = ~np.isnan(kc).all(axis=-1)
    assert written.sum() == T * 4
    assert sorted(kc[written].ravel().tolist()) == sorted(k.ravel().tolist())


def test_write_then_attend_matches_dense_softmax():
    # a prefill (ctx 0) written by write_kv into an empty paged cache, then attended by the
    # paged oracle, equals dense causal softmax attention over the un-paged K/V (Eq. 1/2)
    rng = np.random.default_rng(11)
    hq, hkv, d, bs, L = 4, 2, 16, 16, 45
    q = rng.uniform(-1, 1, (L, hq, d)).astype(np.float32)
    k = rng.uniform(-1, 1, (L, hkv, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (L, hkv, d)).astype(np.float32)
    nb = 6
    bt = np.array([[4, 0, 5, -1]], np.int32)
    cu, sl = np.array([0, L], np.int32), np.array([L], np.int32)
    kc, vc = KV.write_kv(k, v, _nan_cache(nb, bs, hkv, d), _nan_cache(nb, bs, hkv, d), bt, cu, sl, bs)
    scale = 1.0 / np.sqrt(d)
    got = O.paged_attention(q, kc, vc, bt, cu, sl, scale, hkv, bs)
    G = hq // hkv
    for i in range(L):
        for h in range(hq):
            s = (k[: i + 1, h // G].astype(np.float64) @ q[i, h].astype(np.float64)) * scale
            p = np.exp(s - s.max())
            ref = (p[:, None] * v[: i + 1, h // G]).sum(0) / p.sum()
            assert np.allclose(got[i, h], ref, atol=1e-12, rtol=1e-12)
