"""Pins for oracle/softmax.py (tiled softmax P:249-266, segment merge P:367-387) and
oracle/metadata.py against the two-pass C oracle,
closed forms, the paper's worked examples (tests/golden/paper_examples.json) and
brute-force enumeration."""
import json
import math
import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import attention as O
from oracle import metadata as M
from oracle import softmax as S
from workloads import Workload, generate

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def _dense(batch, b):
    w = batch.workload
    L = int(batch.seq_lens[b])
    K = np.stack([O.widen(batch.k_cache)[batch.block_table[b, t // w.block_size], t % w.block_size]
                  for t in range(L)]).astype(np.float64)
    V = np.stack([O.widen(batch.v_cache)[batch.block_table[b, t // w.block_size], t % w.block_size]
                  for t in range(L)]).astype(np.float64)
    return K, V


def _rows_of_seq(batch, b, h):
    w = batch.workload
    s, e = int(batch.cu_seqlens_q[b]), int(batch.cu_seqlens_q[b + 1])
    ctx = int(batch.seq_lens[b]) - (e - s)
    q = O.widen(batch.q)[s:e, h].astype(np.float64)
    vis = [ctx + i + 1 for i in range(e - s)]
    return q, vis, s, e


@settings(max_examples=25, deadline=None)
@given(seed=st.integers(0, 10_000), tile=st.integers(1, 70), nseg=st.integers(1, 9))
def test_tiled_and_segmented_equal_two_pass(seed, tile, nseg):
    w = Workload("t", ((37, 5), (0, 23), (90, 1)), 4, 2, 16, 8, "f32")
    batch = generate(w, seed=seed % 50)
    ref = O.batch_attention(batch)
    for b in range(w.num_seqs):
        K, V = _dense(batch, b)
        for h in (0, 3):
            g = h // 2
            q, vis, s, e = _rows_of_seq(batch, b, h)
            tiles = S.tile_ranges(len(K), tile)
            it = S.finalize(S.tiled_attention(q, K[:, g], V[:, g], w.scale, vis, tiles))
            np.testing.assert_allclose(it, ref[s:e, h], rtol=0, atol=1e-12)
            segs = S.assign_tiles_to_segments(len(tiles), nseg)
            parts = S.segment_partials(q, K[:, g], V[:, g], w.scale, vis, tiles, segs)
            np.testing.assert_allclose(S.merge_segments(parts), ref[s:e, h], rtol=0, atol=1e-12)


def test_fig3_32_tiles_as_4_segments_of_8():
    # 32 tiles processed iteratively == 4 segments x 8 tiles merged
    w = Workload("fig3", ((511, 1),), 8, 1, 64, 16, "bf16")
    batch = generate(w, seed=12, dist="peaked")
    K, V = _dense(batch, 0)
    tiles = S.tile_ranges(512, 16)
    assert len(tiles) == 32
    segs = S.assign_tiles_to_segments(32, 4)
    assert segs == [(0, 8), (8, 16), (16, 24), (24, 32)]
    ref = O.batch_attention(batch)
    for h in range(8):
        q, vis, s, e = _rows_of_seq(batch, 0, h)
        it = S.finalize(S.tiled_attention(q, K[:, 0], V[:, 0], w.scale, vis, tiles))
        mg = S.merge_segments(S.segment_partials(q, K[:, 0], V[:, 0], w.scale, vis, tiles, segs))
        np.testing.assert_allclose(it, ref[s:e, h], rtol=0, atol=1e-12)
        np.testing.assert_allclose(mg, it, rtol=0, atol=1e-12)


def test_merge_identity_permutation_associativity_and_empty_segments():
    rng = np.random.default_rng(3)
    q = rng.uniform(-1, 1, (3, 8))
    K = rng.uniform(-1, 1, (40, 8))
    V = rng.uniform(-1, 1, (40, 8))
    vis = [40, 40, 40]
    tiles = S.tile_ranges(40, 4)
    one = S.segment_partials(q, K, V, 0.3, vis, tiles, [(0, 10)])
    np.testing.assert_allclose(S.merge_segments(one), S.finalize(one[0]), rtol=0, atol=1e-15)
    parts = S.segment_partials(q, K, V, 0.3, vis, tiles, [(0, 3), (3, 7), (7, 10)])
    ref = S.merge_segments(parts)
    np.testing.assert_allclose(S.merge_segments(parts[::-1]), ref, rtol=0, atol=1e-14)
    split = S.segment_partials(q, K, V, 0.3, vis, tiles, [(0, 3), (3, 5), (5, 7), (7, 10)])
    np.testing.assert_allclose(S.merge_segments(split), ref, rtol=0, atol=1e-14)
    segs = S.assign_tiles_to_segments(3, 8)
    parts = S.segment_partials(q, K[:12], V[:12], 0.3, vis, S.tile_ranges(12, 4), segs)
    assert all(not np.isfinite(p[0]).any() and (p[1] == 0).all() for p in parts[3:])
    full = S.finalize(S.tiled_attention(q, K[:12], V[:12], 0.3, [12] * 3, S.tile_ranges(12, 4)))
    np.testing.assert_allclose(S.merge_segments(parts), full, rtol=0, atol=1e-14)


def test_softmax_closed_forms():
    # single key -> its V row; uniform scores -> mean of V; shift invariance; overflow bait
    st0 = S.online_update(S.init_state(1, 2), np.array([[0.3]]), np.array([[1.0, -2.0]]), np.array([[True]]))
    np.testing.assert_array_equal(S.finalize(st0), [[1.0, -2.0]])
    v = np.array([[1.0, 0.0], [3.0, 0.0]])
    st1 = S.online_update(S.init_state(1, 2), np.array([[0.0, 0.0]]), v, np.ones((1, 2), bool))
    np.testing.assert_allclose(S.finalize(st1), [[2.0, 0.0]], rtol=0, atol=1e-15)
    rng = np.random.default_rng(4)
    s = rng.uniform(-3, 3, (2, 9))
    V = rng.uniform(-1, 1, (9, 4))
    a = S.finalize(S.online_update(S.init_state(2, 4), s, V, np.ones((2, 9), bool)))
    b = S.finalize(S.online_update(S.init_state(2, 4), s + 417.0, V, np.ones((2, 9), bool)))
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    big = S.finalize(S.online_update(S.init_state(1, 2), np.array([[1000.0, 1000.0]]), v, np.ones((1, 2), bool)))
    np.testing.assert_allclose(big, [[2.0, 0.0]], rtol=0, atol=1e-15)
    # fully masked tile is a no-op
    st2 = S.online_update(st1, np.array([[5.0, 5.0]]), v * np.nan, np.zeros((1, 2), bool))
    np.testing.assert_array_equal(S.finalize(st2), S.finalize(st1))


# ---------------------------------------------------------------- metadata

def test_golden_q_blocks_and_batch_meta():
    for ex in GOLDEN["q_blocks"]:
        m = M.build_batch_meta([0, ex["query_len"]], [ex["query_len"]], ex["block_q"])
        assert m["num_q_blocks"][0] == ex["num_q_blocks"], ex["cite"]
    for ex in GOLDEN["batch_meta"]:
        m = M.build_batch_meta(ex["cu_seqlens_q"], ex["seq_lens"], ex["block_q"])
        assert m["cu_q_blocks"].tolist() == ex["cu_q_blocks"], ex["cite"]


def test_golden_lookup_headmap_slots_segments():
    for ex in GOLDEN["seq_lookup"]:
        assert M.seq_index_lookup(ex["cu"], ex["idx"]) == ex["seq"], ex["cite"]
    for ex in GOLDEN["head_map"]:
        assert M.kv_head_for_query_head(ex["q_head"], ex["num_q_heads"], ex["num_kv_heads"]) == ex["kv_head"]
    ex = GOLDEN["paged_slot"][0]
    row = list(range(100, 110))
    assert M.paged_slot(row, ex["t"], ex["block_size"]) == (row[ex["table_index"]], ex["slot"])
    ex = GOLDEN["paged_slot"][1]
    assert -(-ex["seq_len"] // ex["block_size"]) == ex["num_blocks"]
    for ex in GOLDEN["segments"]:
        got = S.assign_tiles_to_segments(ex["num_tiles"], ex["num_segments"])
        assert [list(r) for r in got] == ex["ranges"], ex["cite"]


def test_qblock_count_random_pairs_bruteforce():
    rng = np.random.default_rng(5)
    for _ in range(1000):
        q = int(rng.integers(1, 5000))
        bq = int(rng.integers(1, 129))
        m = M.build_batch_meta([0, q], [q], bq)
        # brute force: count blocks by walking tokens
        n, t = 0, 0
        while t < q:
            n += 1
            t += bq
        assert m["num_q_blocks"][0] == n == math.ceil(q / bq)


def test_token_partition_and_decode_count():
    rng = np.random.default_rng(6)
    for _ in range(50):
        B = int(rng.integers(1, 12))
        qs = rng.integers(0, 9, size=B)
        cu = np.concatenate([[0], np.cumsum(qs)])
        sl = qs + rng.integers(0, 50, size=B)
        m = M.build_batch_meta(cu, sl, 4)
        if cu[-1] == 0:
            continue
        owners = [M.seq_index_lookup(cu, t) for t in range(int(cu[-1]))]
        assert np.bincount(owners, minlength=B).tolist() == qs.tolist()
        assert m["num_decodes"] == int((qs == 1).sum())
        qb_owner = [M.seq_index_lookup(m["cu_q_blocks"], j) for j in range(m["total_q_blocks"])]
        assert np.bincount(qb_owner, minlength=B).tolist() == [(-(-q // 4)) for q in qs]


def test_errors():
    with pytest.raises(ValueError):
        M.build_batch_meta([0, 5], [3], 2)
    with pytest.raises(IndexError):
        M.seq_index_lookup([0, 3], 3)
    with pytest.raises(IndexError):
        M.kv_head_for_query_head(32, 32, 8)
    with pytest.raises(ValueError):
        S.assign_tiles_to_segments(4, 0)


def test_qblock_rows_token_major():
    rows = M.qblock_rows(2, 2, 5, 1, 4)  # q_len 5, BLOCK_Q 2 -> third block holds token 4 only
    assert rows == [(4, 4), (4, 5), (4, 6), (4, 7)]
