"""Tuning flow (§4.2; SPEC tuner S:375-463): the regret-minimising tree
fitter, its JSON/array forms, and libpattn's consultation of an installed tree
(pattn_set_tuning_tree / pattn_plan_tuning are host-only, so this runs on CPU)."""
import os

import numpy as np
import pytest

from paper_2511_11581_b200 import tuner

A = {"items_per_sm": 0, "min_chunk_tokens": 0, "decode_ctas_per_sm": 2, "k2_sm_mbs": 0, "serial": 0,
     "decode_kernel": 1}  # = libpattn's built-in defaults
B = {"items_per_sm": 4, "min_chunk_tokens": 1024, "decode_ctas_per_sm": 3, "k2_sm_mbs": 80000, "serial": 0,
     "decode_kernel": 2}
C = {"items_per_sm": 32, "min_chunk_tokens": 64, "decode_ctas_per_sm": 1, "k2_sm_mbs": 45000, "serial": 1,
     "decode_kernel": 1}


def _rec(label, feats, cfg, mean):
    return {"scenario": label, "features": feats, "config": cfg, "latency_us": {"mean": mean, "p50": mean, "p95": mean}}


def _feats(seqs, tokens, maxq, maxl):
    return {"num_seqs": seqs, "num_tokens": tokens, "max_query_len": maxq, "max_seq_len": maxl}


def test_single_best_config_gives_depth0_tree():
    recs = []
    for i, f in enumerate([_feats(8, 8, 1, 4096), _feats(64, 16440, 2048, 4097), _feats(1, 1, 1, 131073)]):
        recs += [_rec(f"s{i}", f, A, 10.0 + i), _rec(f"s{i}", f, B, 20.0 + i)]
    tree = tuner.fit_decision_tree(recs, max_depth=3)
    assert tuner.depth(tree) == 0 and tuner.select(tree, _feats(5, 5, 5, 5)) == A


def test_decode_only_vs_prefill_split_on_max_query_len():
    # decode-only scenarios (max_query_len 1) prefer B, the others prefer A -> one split on max_query_len
    recs = []
    for i, (maxq, best, ns) in enumerate([(1, B, 16), (1, B, 64), (2048, A, 32), (512, A, 8)]):
        f = _feats(ns, ns if maxq == 1 else 4096, maxq, 8192)  # num_seqs does not separate the classes
        other = A if best is B else B
        recs += [_rec(f"s{i}", f, best, 100.0), _rec(f"s{i}", f, other, 130.0)]
    tree = tuner.fit_decision_tree(recs, max_depth=3)
    assert tuner.depth(tree) == 1 and tree["feature"] in ("max_query_len", "num_tokens")
    assert tuner.select(tree, _feats(3, 3, 1, 100)) == B
    assert tuner.select(tree, _feats(3, 9000, 2048, 100)) == A
    assert tuner.tree_regret(tree, recs) == 0.0


def test_min_gain_suppresses_noise_splits():
    # two scenario classes whose best configs differ by 0.3 % (noise-level) vs 30 %: with a 1 %
    # noise floor only the large difference may split the tree
    def recs(gap):
        out = []
        for i, (maxq, best, ns) in enumerate([(1, B, 16), (1, B, 64), (2048, A, 32), (512, A, 8)]):
            f = _feats(ns, ns if maxq == 1 else 4096, maxq, 8192)
            other = A if best is B else B
            out += [_rec(f"s{i}", f, best, 100.0), _rec(f"s{i}", f, other, 100.0 + gap)]
        return out
    assert tuner.depth(tuner.fit_decision_tree(recs(0.3), max_depth=3)) == 1  # unregularised: splits
    assert tuner.depth(tuner.fit_decision_tree(recs(0.3), max_depth=3, min_gain=0.01)) == 0
    assert tuner.depth(tuner.fit_decision_tree(recs(30.0), max_depth=3, min_gain=0.01)) == 1


def test_tree_regret_never_worse_than_best_global_config():
    rng = np.random.default_rng(0)
    recs = []
    for i in range(40):
        f = _feats(int(rng.integers(1, 300)), int(rng.integers(1, 70000)), int(rng.choice([1, 16, 2048])),
                   int(rng.integers(16, 140000)))
        for cfg in (A, B, C):
            recs.append(_rec(f"s{i}", f, cfg, float(rng.uniform(10, 100))))
    for d in (0, 1, 2, 4):
        tree = tuner.fit_decision_tree(recs, max_depth=d)
        assert tuner.depth(tree) <= d
        assert tuner.tree_regret(tree, recs) <= tuner.best_global_regret(recs) + 1e-9
    # total: any feature vector reaches a leaf; flattened array children come after parents
    for _ in range(200):
        f = _feats(*[int(x) for x in rng.integers(0, 200000, 4)])
        assert set(tuner.select(tree, f)) == set(tuner.KNOBS)
    nodes = tuner.flatten(tree)
    for i, n in enumerate(nodes):
        if n.feature >= 0:
            assert i < n.lt < len(nodes) and i < n.ge < len(nodes)


def test_empty_records_raise():
    with pytest.raises(tuner.NoData):
        tuner.fit_decision_tree([])


def test_records_roundtrip(tmp_path):
    p = str(tmp_path / "r.ndjson")
    recs = [_rec("x", _feats(1, 1, 1, 1), A, 3.0)]
    tuner.write_records(p, recs)
    back = tuner.read_records(p)
    assert back[0]["v"] == 1 and back[0]["config"] == A


def _problem(lib, B=64, T=64, maxq=1, maxl=4097):
    p = lib.Problem()
    p.num_seqs, p.num_tokens, p.num_q_heads, p.num_kv_heads, p.head_dim = B, T, 32, 8, 128
    p.block_size, p.num_blocks, p.max_blocks_per_seq, p.dtype = 16, 16448, 257, 1
    p.max_query_len, p.max_seq_len = maxq, maxl
    p.q_stride_tok, p.q_stride_head = 32 * 128, 128
    p.kv_stride_blk, p.kv_stride_tok, p.kv_stride_head = 16 * 8 * 128, 8 * 128, 128
    p.bt_stride = 257
    p.o_stride_tok, p.o_stride_head = 32 * 128, 128
    return p


def test_committed_tree_is_valid_and_installed():
    from paper_2511_11581_b200 import pattn

    tree = tuner.default_tree()
    assert tree is not None and tuner.depth(tree) <= 6
    pattn.load()
    # config 3's shape resolves to the tree's leaf (no env overrides in the test environment)
    p = _problem(pattn, maxq=2048, T=16440)
    if not any(os.environ.get(k) for k in ("PATTN_ITEMS_PER_SM", "PATTN_MIN_CHUNK_TOKENS", "PATTN_DECODE_CTAS",
                                           "PATTN_K2_SM_GBS", "PATTN_SERIAL")):
        assert tuner.planned_tuning(p) == tuner.with_defaults(tuner.select(
            tree, {"num_seqs": 64, "num_tokens": 16440, "max_query_len": 2048, "max_seq_len": 4097}))


def test_libpattn_consults_installed_tree(monkeypatch):
    from paper_2511_11581_b200 import pattn

    for k in ("PATTN_ITEMS_PER_SM", "PATTN_MIN_CHUNK_TOKENS", "PATTN_DECODE_CTAS", "PATTN_K2_SM_GBS", "PATTN_SERIAL"):
        monkeypatch.delenv(k, raising=False)
    tree = {"feature": "max_query_len", "threshold": 1.5, "lt": B,
            "ge": {"feature": "num_seqs", "threshold": 100, "lt": A, "ge": C}}
    try:
        tuner.install(None)
        assert tuner.planned_tuning(_problem(pattn)) == A  # built-in defaults
        tuner.install(tree)
        assert tuner.planned_tuning(_problem(pattn)) == B
        assert tuner.planned_tuning(_problem(pattn, maxq=2048, T=16440)) == A
        assert tuner.planned_tuning(_problem(pattn, B=256, maxq=2048, T=65760)) == C
        monkeypatch.setenv("PATTN_DECODE_CTAS", "4")  # environment overrides win
        assert tuner.planned_tuning(_problem(pattn))["decode_ctas_per_sm"] == 4
        monkeypatch.delenv("PATTN_DECODE_CTAS")
        # malformed trees are rejected and the installed one stays
        bad = tuner.flatten(tree)
        bad[0].lt = 0  # child index not after its parent (a cycle)
        arr = (tuner.TreeNode * len(bad))(*bad)
        assert pattn.load().pattn_set_tuning_tree(arr, len(bad)) == 1
        bad2 = tuner.flatten({"items_per_sm": 1, "min_chunk_tokens": 1, "decode_ctas_per_sm": 9})
        arr2 = (tuner.TreeNode * 1)(*bad2)
        assert pattn.load().pattn_set_tuning_tree(arr2, 1) == 1
        bad3 = tuner.flatten(dict(A, serial=2))  # serial is 0 or 1
        assert pattn.load().pattn_set_tuning_tree((tuner.TreeNode * 1)(*bad3), 1) == 1
        assert tuner.planned_tuning(_problem(pattn)) == B
    finally:
        tuner.install(tuner.default_tree())  # what pattn.load() installs
