"""GPU parity: libpattn (through its C ABI) vs the fp64 oracle, element by element, on the
same seeded inputs (workloads/).  Tolerances from north_star: bf16 |err| <= 1e-2 + 1e-2|ref|,
fp32 |err| <= 1e-5 + 1e-5|ref|; indexing bit-exact (needle tests, debug_plan)."""
import os

import numpy as np
import pytest
import torch

from oracle import attention as O
from oracle import metadata as M
from workloads import CONFIGS, Workload, generate
from workloads.gen import random_workload

from gpu_helpers import DeviceBatch, assert_close, out_f64

pytestmark = pytest.mark.gpu

P = None


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    global P
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_11581_b200 import pattn

    pattn.load()
    P = pattn


def _check(batch, flags=0, what=""):
    ref = O.batch_attention(batch)
    db = DeviceBatch(batch)
    gpu = out_f64(db.run(flags=flags))
    return assert_close(gpu, ref, batch.dtype, what or batch.workload.name)


# ---------------------------------------------------------------- config 1 (fp32)
@pytest.mark.parametrize("layout", ["NHD", "HND"])
def test_config1_fp32(layout):
    batch = generate(CONFIGS["c1_tiny"], seed=1001, layout=layout)
    _check(batch)


def test_config1_as_bf16_all_paths():
    w = CONFIGS["c1_tiny"]
    wb = Workload("c1_bf16", w.seqs, w.num_q_heads, w.num_kv_heads, w.head_dim, w.block_size, "bf16")
    batch = generate(wb, seed=1001)
    for flags in (0, P.FLAG_FORCE_GENERIC, P.FLAG_NO_SPLIT, P.FLAG_FORCE_SPLIT):
        _check(batch, flags, f"c1 bf16 flags={flags}")


# ---------------------------------------------------------------- random mixed batches
CASES = [
    # heads, D, bs, dtype, layout, dist
    ((32, 8), 128, 16, "bf16", "NHD", "uniform"),
    ((32, 8), 128, 16, "bf16", "NHD", "peaked"),
    ((64, 8), 128, 16, "bf16", "HND", "peaked"),
    ((16, 1), 128, 32, "bf16", "NHD", "peaked"),
    ((8, 8), 64, 16, "bf16", "NHD", "peaked"),
    ((12, 2), 128, 80, "bf16", "NHD", "peaked"),   # bs 80 (hybrid-model block size)
    ((4, 1), 64, 7, "bf16", "HND", "peaked"),      # bs not a multiple of 16 -> generic path
    ((32, 8), 128, 16, "f32", "NHD", "peaked"),
    ((16, 1), 64, 5, "f32", "HND", "uniform"),
    ((128, 2), 128, 16, "bf16", "NHD", "peaked"),  # G = 64
    ((32, 8), 128, 80, "bf16", "NHD", "peaked"),   # bs 80 on the tcgen05 prefill path (G = 4)
    ((64, 8), 128, 48, "bf16", "HND", "peaked"),   # bs 48: 3 sub-blocks per paged block, G = 8
    ((8, 8), 128, 128, "bf16", "NHD", "peaked"),   # bs 128, G = 1 (BLOCK_Q = 256 tokens)
    ((32, 8), 128, 16, "f16", "NHD", "peaked"),    # fp16 storage: K1 / K2 / K3 with f16 operands
    ((64, 8), 128, 80, "f16", "HND", "uniform"),
    ((8, 8), 64, 7, "f16", "NHD", "peaked"),       # fp16, bs 7: K4 with split decodes
]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("seed", [0, 1])
def test_random_mixed(case, seed):
    heads, D, bs, dt, layout, dist = CASES[case]
    rng = np.random.default_rng(1000 * case + seed)
    w = random_workload(rng, heads, D, bs, dt, max_seqs=6, max_len=700, decode_share=0.5)
    batch = generate(w, seed=seed, dist=dist, layout=layout)
    _check(batch, 0, f"case {case} {w.seqs}")
    if dt == "bf16":
        _check(batch, P.FLAG_FORCE_SPLIT, f"case {case} force-split")


@pytest.mark.parametrize("flags", [0, 0x1, 0x2, 0x4])
def test_long_decode_split(flags):
    w = Workload("longdec", ((5000, 1), (3000, 1), (17, 1), (0, 1), (1, 1)), 64, 8, 128, 16, "bf16")
    batch = generate(w, seed=5, dist="peaked")
    _check(batch, flags, f"long decode flags={flags}")


PREFILL_CASES = [
    # (seqs, heads, bs, layout)
    (((0, 1000), (2000, 300), (0, 129), (77, 1)), (32, 8), 16, "NHD"),
    (((0, 777), (130, 260)), (64, 8), 16, "NHD"),
    (((0, 515), (1000, 64)), (32, 8), 64, "HND"),
    (((3, 200), (0, 47)), (16, 1), 32, "NHD"),
    (((0, 300),), (8, 8), 16, "NHD"),       # G = 1: BLOCK_Q = 128
    (((0, 257), (9, 9)), (128, 2), 128, "NHD"),  # G = 64: BLOCK_Q = 2; bs 128 = one block per tile
    # G not dividing 128 (common GQA ratios): BLOCK_Q = 2 * floor(128 / G), padding rows per half
    (((0, 700), (300, 90), (5, 1)), (48, 8), 16, "NHD"),   # G = 6 (21 tokens x 6 = 126 rows per half)
    (((0, 500), (64, 130)), (28, 4), 16, "HND"),           # G = 7 (Qwen-style 28q/4kv)
    (((0, 333), (17, 40)), (96, 8), 32, "NHD"),            # G = 12 (10 tokens x 12 = 120 rows)
    (((0, 290),), (15, 5), 16, "NHD"),                     # G = 3 (42 x 3 = 126)
    (((0, 260), (100, 33)), (40, 8), 48, "NHD"),           # G = 5 (25 x 5 = 125)
]


@pytest.mark.parametrize("case", range(len(PREFILL_CASES)))
def test_prefill_tensor_core_path(case):
    seqs, heads, bs, layout = PREFILL_CASES[case]
    w = Workload(f"prefill{case}", seqs, heads[0], heads[1], 128, bs, "bf16")
    kv = np.zeros((1, bs, heads[1], 128), np.uint16)
    p = P.make_problem(torch.zeros((1, heads[0], 128), dtype=torch.bfloat16, device="cuda"),
                       torch.zeros(kv.shape, dtype=torch.bfloat16, device="cuda"), heads[1], bs,
                       torch.zeros((1, 1), dtype=torch.int32, device="cuda"), 1, max_query_len=64)
    assert P.planned_kernels(p) & (1 << P.KERNEL_PREFILL), "not on the tcgen05 prefill kernel"  # K1, not K4
    batch = generate(w, seed=100 + case, dist="peaked", layout=layout)
    _check(batch, 0, f"prefill case {case}")


@pytest.mark.parametrize("heads,bs,layout", [((8, 8), 16, "NHD"), ((32, 8), 16, "HND"), ((28, 4), 32, "NHD"),
                                              ((64, 8), 80, "NHD"), ((16, 1), 16, "NHD")])
def test_prefill_tensor_core_path_head_dim_64(heads, bs, layout):
    """bf16 head_dim 64 on the tcgen05 prefill kernel (K1 instantiated for D = 64)."""
    w = Workload("prefill_d64", ((0, 700), (300, 90), (0, 65), (5, 1), (1000, 1)), heads[0], heads[1], 64, bs, "bf16")
    batch = generate(w, seed=61, dist="peaked", layout=layout, poison=True)
    db = DeviceBatch(batch)
    p = P.make_problem(db.q, db.k, heads[1], bs, db.bt, w.num_seqs, None, layout, 700, 1001)
    assert P.planned_kernels(p) & (1 << P.KERNEL_PREFILL)
    _check(batch, 0, f"prefill d64 {heads} bs={bs}")


def test_chunked_prefill_and_empty_sequences():
    w = Workload("chunked", ((300, 40), (0, 0), (77, 1), (5, 129), (0, 0), (0, 33)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=6, dist="peaked")
    _check(batch, 0, "chunked")


# ---------------------------------------------------------------- bit-exact indexing
@pytest.mark.parametrize("flags", [0, 0x1, 0x4])
def test_needle_bit_exact(flags):
    w = Workload("needle", ((700, 1), (0, 50), (1500, 1), (40, 20), (33, 1)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=7, dist="needle")
    db = DeviceBatch(batch)
    out = db.run(flags=flags).cpu()
    v = O.widen(batch.v_cache)
    for b in range(w.num_seqs):
        s, e = int(batch.cu_seqlens_q[b]), int(batch.cu_seqlens_q[b + 1])
        for g in range(w.num_kv_heads):
            t = int(batch.needle_pos[b, g])
            row = torch.from_numpy(v[batch.block_table[b, t // 16], t % 16, g]).to(torch.bfloat16)
            for h in range(g * 4, g * 4 + 4):
                got = out[s:e, h]
                assert torch.equal(got, row.expand_as(got)), (b, g, h, t)


def test_needle_sweep_positions_decode():
    # needle at every block boundary class of a split decode sequence: first/last slot, segment edges
    L = 4097
    for t in (0, 15, 16, 2047, 2048, 4095, 4096):
        w = Workload("nsweep", ((L - 1, 1),), 32, 8, 128, 16, "bf16")
        batch = generate(w, seed=8, dist="needle", needle_pos=[[t] * 8])
        out = DeviceBatch(batch).run(flags=0x4).cpu()
        v = O.widen(batch.v_cache)
        row = torch.from_numpy(v[batch.block_table[0, t // 16], t % 16, 3]).to(torch.bfloat16)
        assert torch.equal(out[0, 12], row), t


def test_debug_plan_bit_exact():
    rng = np.random.default_rng(9)
    for trial in range(10):
        w = random_workload(rng, (32, 8), 128, 16, "bf16", max_seqs=40, max_len=3000, decode_share=0.6)
        batch = generate(w, seed=trial, poison=False)
        db = DeviceBatch(batch)
        for flags in (0, P.FLAG_FORCE_GENERIC, P.FLAG_FORCE_SPLIT):
            prob = P.make_problem(db.q, db.k, w.num_kv_heads, w.block_size, db.bt, w.num_seqs, flags=flags)
            plan = P.debug_plan(prob, db.cu, db.sl).cpu().numpy()
            B = w.num_seqs
            block_q = int(plan[3])
            qlens = np.diff(batch.cu_seqlens_q)
            dec = qlens == 1  # decode units on K2, or split on K4 (FORCE_GENERIC)
            # Q-block kernel sequences: everything not routed to the decode kernel
            cu_qb_ref = M.build_batch_meta(np.concatenate([[0], np.cumsum(np.where(dec, 0, qlens))]),
                                           np.where(dec, 0, batch.seq_lens), block_q)["cu_q_blocks"]
            assert plan[8:8 + B + 1].tolist() == cu_qb_ref.tolist()
            assert plan[0] == cu_qb_ref[-1]
            assert plan[1] == int(dec.sum())
            cu_ch = plan[8 + B + 1: 8 + 2 * B + 2]
            nch = np.diff(cu_ch)
            C = int(plan[4])
            nblk = (batch.seq_lens + 15) // 16
            exp = np.where(dec, -(-nblk // C), 0)
            assert nch.tolist() == exp.tolist()
            assert plan[2] == cu_ch[-1]


# ---------------------------------------------------------------- robustness
def test_poison_canary_and_determinism():
    w = Workload("canary", ((900, 1), (0, 64), (20, 9), (4000, 1)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=10, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    T, Hq, D = db.q.shape
    big = torch.full((T + 3, Hq, D), 1234.5, dtype=torch.bfloat16, device="cuda")
    o1 = db.run(out=big[:T]).clone()
    assert torch.all(big[T:] == 1234.5)
    assert torch.isfinite(o1.float()).all()
    o2 = db.run()
    assert torch.equal(o1, o2)
    ref = O.batch_attention(batch)
    assert_close(out_f64(o1), ref, "bf16", "canary")


def test_hostio_equals_device_path():
    w = Workload("hostio", ((100, 1), (0, 48), (2000, 1)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=11, dist="peaked")
    db = DeviceBatch(batch)
    dev = db.run().cpu()
    q_h = db.q.cpu().pin_memory()
    out_h = torch.empty_like(q_h).pin_memory()
    P.unified_attention_hostio(q_h, db.k, db.v, db.bt.cpu().pin_memory(), db.cu.cpu().pin_memory(),
                               db.sl.cpu().pin_memory(), w.scale, w.num_kv_heads, w.block_size, out_h,
                               max_query_len=48, max_seq_len=2001)
    torch.cuda.synchronize()
    assert torch.equal(out_h, dev)


def test_two_stream_equals_serial():
    w = Workload("streams", tuple([(0, 200)] * 2 + [(1000, 1)] * 6), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=12, dist="peaked")
    db = DeviceBatch(batch)
    a = db.run().clone()
    s2 = torch.cuda.Stream()
    b = db.run(stream2=s2)
    assert torch.equal(a, b)


def test_dynamic_scheduling_is_bitwise_deterministic():
    """Work items are claimed from global counters, so the item -> CTA mapping changes from run to
    run (and with two streams); every item's arithmetic must not depend on it."""
    seqs = tuple([(3000 + 37 * i, 1) for i in range(96)] + [(200 * i, 300 + 50 * i) for i in range(6)])
    w = Workload("dyn", seqs, 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=15, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    a = db.run().clone()
    s2 = torch.cuda.Stream()
    for i in range(6):
        b = db.run(stream2=s2) if i % 2 else db.run()
        assert torch.equal(a, b), f"run {i}"


def test_cuda_graph_capture_and_replay_with_new_metadata():
    """The call is sync-free with data-independent grids (static launch grid), so it can
    be captured once and replayed with different device-resident metadata."""
    w = Workload("graph", ((100, 50), (2000, 1), (0, 30), (700, 1), (33, 64)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=14, dist="peaked")
    db = DeviceBatch(batch)
    # metadata A: sequences 0 and 2 swapped (same T, same table width) -- used only for capture
    order = [2, 1, 0, 3, 4]
    qlens = np.diff(batch.cu_seqlens_q)
    cu_a = np.concatenate([[0], np.cumsum(qlens[order])]).astype(np.int32)
    sl_a = batch.seq_lens[order].astype(np.int32)
    bt_a = batch.block_table[order].astype(np.int32)
    cu_b, sl_b, bt_b = db.cu.clone(), db.sl.clone(), db.bt.clone()
    db.cu.copy_(torch.from_numpy(cu_a))
    db.sl.copy_(torch.from_numpy(sl_a))
    db.bt.copy_(torch.from_numpy(bt_a))
    out = torch.empty_like(db.q)
    s = torch.cuda.Stream()
    kw = dict(max_query_len=64, max_seq_len=2001, stream=s)
    with torch.cuda.stream(s):
        P.unified_attention(db.q, db.k, db.v, db.bt, db.cu, db.sl, w.scale, 8, 16, out, **kw)  # warm-up
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        P.unified_attention(db.q, db.k, db.v, db.bt, db.cu, db.sl, w.scale, 8, 16, out, **kw)
    db.cu.copy_(cu_b)
    db.sl.copy_(sl_b)
    db.bt.copy_(bt_b)
    out.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    assert_close(out_f64(out), O.batch_attention(batch), "bf16", "graph replay")


def test_error_codes():
    w = CONFIGS["c1_tiny"]
    batch = generate(w, seed=13)
    db = DeviceBatch(batch)
    with pytest.raises(P.PattnError) as ei:
        P.unified_attention(db.q, db.k, db.v, db.bt, db.cu, db.sl, w.scale, w.num_kv_heads, w.block_size,
                            workspace=torch.empty(16, dtype=torch.uint8, device="cuda"))
    assert ei.value.code == 6


# ---------------------------------------------------------------- BASELINE.json full sizes (sampled rows)
def _sample_rows(batch, n_random, rng):
    w = batch.workload
    rows = []
    qlens = np.diff(batch.cu_seqlens_q)
    for b in range(w.num_seqs):
        s = int(batch.cu_seqlens_q[b])
        if qlens[b] == 1:
            rows += [s * w.num_q_heads + h for h in range(w.num_q_heads)]
        elif qlens[b] > 1:
            for tok in (s, s + int(qlens[b]) - 1):
                rows += [tok * w.num_q_heads + h for h in range(w.num_q_heads)]
    T = w.num_tokens
    rows += rng.integers(0, T * w.num_q_heads, size=n_random).tolist()
    return np.unique(np.array(rows, np.int64))


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2_decode8b", "c3_mixed8b", "c4_decode128k", "c5_mixed70b", "x_bs7_mixed"])
def test_full_size_sampled(name):
    from workloads.gen import ATTRIBUTION

    w = CONFIGS[name] if name in CONFIGS else ATTRIBUTION[name]
    batch = generate(w, seed=2000 + (list(CONFIGS) + list(ATTRIBUTION)).index(name), dist="peaked", poison=True)
    db = DeviceBatch(batch)
    o_serial = db.run()
    if any(q > 1 for _, q in w.seqs):
        # bench's launch configuration: decode kernels on a second stream over K5's SM split;
        # per-item arithmetic is unchanged, so the output must be bitwise the serial one
        o_two = db.run(stream2=torch.cuda.Stream())
        assert torch.equal(o_two, o_serial), name
    out = out_f64(o_serial).reshape(-1, w.head_dim)
    rows = _sample_rows(batch, 2000, np.random.default_rng(3))
    ref = O.batch_attention(batch, rows=rows)
    assert_close(out[rows], ref, w.dtype, name)


@pytest.mark.slow
def test_compute_sanitizer_memcheck_and_racecheck():
    """compute-sanitizer on a small mixed batch through the C ABI (prefill + split decode)."""
    import os
    import shutil
    import subprocess

    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = os.path.join(root, "scripts", "one_call.py")
    for tool, seqs in (("memcheck", "6x3000:1+2x0:300+1x50:70"), ("racecheck", "2x700:1+1x0:200"), ("synccheck", "2x700:1+1x0:200")):
        r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "3", "python", script, "c3_mixed8b", "1", seqs],
                           capture_output=True, text=True, timeout=900)
        if "ERROR SUMMARY" not in r.stdout and "closed on this pool" in (r.stdout + r.stderr):
            pytest.skip("compute-sanitizer is disabled on this GPU pool")
        # the only accepted report is torch's own benign cuKernelGetFunction probe
        errs = [l for l in r.stdout.splitlines() if "ERROR SUMMARY" in l]
        assert r.returncode in (0, 3), r.stdout[-2000:] + r.stderr[-2000:]
        bad = [l for l in r.stdout.splitlines() if "Program hit" in l and "cuKernelGetFunction" not in l]
        hazards = [l for l in r.stdout.splitlines() if "RACECHECK SUMMARY" in l and " 0 hazards" not in l]
        assert not bad and not hazards, (tool, errs, bad, hazards, r.stdout[-3000:])
        assert "ok c3_mixed8b" in r.stdout, r.stdout[-2000:]


def test_strided_out_and_q_canary():
    """q and out as head-slices of wider tensors (token stride (Hq+2)*D): the TMA-store epilogue
    and every other writer must honour the strides and leave the two extra heads untouched."""
    w = Workload("strided", ((0, 200), (700, 1), (16, 48), (3000, 1)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=12, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    T, Hq, D = db.q.shape
    qw = torch.zeros((T, Hq + 2, D), dtype=torch.bfloat16, device="cuda")
    qw[:, 1:Hq + 1] = db.q
    ow = torch.full((T, Hq + 2, D), 777.0, dtype=torch.bfloat16, device="cuda")
    db.q = qw[:, 1:Hq + 1]
    o = db.run(out=ow[:, 1:Hq + 1])
    assert torch.all(ow[:, 0] == 777.0) and torch.all(ow[:, Hq + 1] == 777.0)
    assert_close(out_f64(o), O.batch_attention(batch), "bf16", "strided")


@pytest.mark.parametrize("flags", [0, 0x4])
def test_segment_reduce_groups_follow_segment_count(flags):
    """K3 on sequences from 1 to several hundred segments in one batch (one warp per (sequence,
    head) item, or eight for long contexts / forced splitting), against the oracle, and bitwise
    reproducible."""
    w = Workload("k3groups", ((20000, 1), (0, 40), (3000, 1), (17, 1), (9000, 1), (60000, 1)), 64, 8, 128, 16,
                 "bf16")
    batch = generate(w, seed=13, dist="peaked")
    ref = O.batch_attention(batch)
    db = DeviceBatch(batch)
    a = db.run(flags=flags).clone()
    assert_close(out_f64(a), ref, "bf16", f"K3 groups flags={flags}")
    assert torch.equal(db.run(flags=flags), a)


@pytest.mark.parametrize("dt,bs,layout", [("bf16", 7, "NHD"), ("f32", 16, "HND"), ("f32", 5, "NHD"), ("bf16", 24, "HND")])
@pytest.mark.parametrize("flags", [0, 0x4])
def test_split_decode_on_generic_path(dt, bs, layout, flags, monkeypatch):
    """Block sizes the TMA decode cannot fetch (not a multiple of 16) and the fp32 path: decodes
    still run as split-KV segments (parallel tiled softmax) -- on the SIMT kernel K4
    (bf16 here with the gathered K2W switched off: decode_kernel 2) -- and K3 merges them; long
    contexts get many segments."""
    monkeypatch.setenv("PATTN_DECODE_WIDE", "0")
    monkeypatch.setenv("PATTN_DISABLE_K1", "1")  # the prefills too (K1 gathers rows for such block sizes)
    w = Workload("k4split", ((20000, 1), (0, 70), (3000, 1), (17, 1), (700, 40), (9000, 1)), 32, 8, 128, bs, dt)
    batch = generate(w, seed=17, dist="peaked", poison=True, layout=layout)
    db = DeviceBatch(batch)
    p = P.make_problem(db.q, db.k, w.num_kv_heads, w.block_size, db.bt, w.num_seqs, None, layout, 70, 20001, flags)
    assert P.planned_kernels(p) == (1 << P.KERNEL_METADATA) | (1 << P.KERNEL_GENERIC) | (1 << P.KERNEL_REDUCE)
    plan = P.debug_plan(p, db.cu, db.sl).cpu().numpy()
    B = w.num_seqs
    nch = np.diff(plan[8 + B + 1: 8 + 2 * B + 2])
    assert nch[0] > 1  # the 20k-token decode is split
    a = db.run(flags=flags).clone()
    assert_close(out_f64(a), O.batch_attention(batch), dt, f"K4 split decode {dt} bs={bs} flags={flags}")
    assert torch.equal(db.run(flags=flags), a)


def test_fp16_tensor_core_paths_and_needle():
    """fp16 storage (PATTN_DTYPE_F16) runs the same kernels as bf16 with f16 UMMA / mma.sync
    operands: the tcgen05 prefill and the TMA decode are planned, the output matches the oracle,
    and the needle case is bit-exact (P = 1 for the needle, exactly 0 elsewhere)."""
    w = Workload("f16mix", ((0, 700), (5000, 1), (300, 90), (20000, 1), (9, 1)), 32, 8, 128, 16, "f16")
    batch = generate(w, seed=51, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    p = P.make_problem(db.q, db.k, 8, 16, db.bt, w.num_seqs, None, "NHD", 700, 20001)
    assert P.planned_kernels(p) & (1 << P.KERNEL_PREFILL) and P.planned_kernels(p) & (1 << P.KERNEL_DECODE)
    _check(batch, 0, "fp16 mixed")
    _check(batch, P.FLAG_FORCE_SPLIT, "fp16 forced split")
    wn = Workload("f16needle", ((700, 1), (0, 50), (1500, 1), (40, 20)), 32, 8, 128, 16, "f16")
    nb = generate(wn, seed=7, dist="needle")
    out = DeviceBatch(nb).run().cpu()
    v = nb.v_cache
    for b in range(wn.num_seqs):
        s_, e_ = int(nb.cu_seqlens_q[b]), int(nb.cu_seqlens_q[b + 1])
        for g in range(wn.num_kv_heads):
            t = int(nb.needle_pos[b, g])
            row = torch.from_numpy(np.ascontiguousarray(v[nb.block_table[b, t // 16], t % 16, g]))
            for tok in range(s_, e_):
                for h in range(g * 4, g * 4 + 4):
                    assert torch.equal(out[tok, h], row), (b, g, tok, h)


def test_hintless_call_matches_oracle():
    """No host hints (max_query_len / max_seq_len = 0): the planner uses its upper bounds."""
    w = Workload("nohint", ((0, 300), (2500, 1), (64, 40), (900, 1)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=21, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    o = P.unified_attention(db.q, db.k, db.v, db.bt, db.cu, db.sl, w.scale, w.num_kv_heads, w.block_size)
    torch.cuda.synchronize()
    assert_close(out_f64(o), O.batch_attention(batch), "bf16", "hint-less")


def test_hint_violation_detected_in_debug_mode(monkeypatch):
    """A max_query_len hint below the true maximum drops the Q-block kernel from the plan; with
    PATTN_DEBUG_SYNC=1 the call synchronises and reports it (PATTN_ERR_INVALID_SEQUENCE)."""
    import subprocess
    import sys

    code = r"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2511_11581_b200 import pattn as P
from workloads import Workload, generate
from gpu_helpers import DeviceBatch
w = Workload("viol", ((0, 50), (700, 1)), 32, 8, 128, 16, "bf16")
db = DeviceBatch(generate(w, seed=3))
try:
    P.unified_attention(db.q, db.k, db.v, db.bt, db.cu, db.sl, w.scale, 8, 16, max_query_len=1, max_seq_len=701)
    print("no error")
except P.PattnError as e:
    print("code", e.code)
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PATTN_DEBUG_SYNC="1", PYTHONPATH=os.path.join(root, "tests"))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert "code 3" in r.stdout, r.stdout + r.stderr[-2000:]


def test_binding_rejects_mismatched_tensors():
    """the binding checks what raw pointers cannot carry (V vs K strides, out vs q,
    int32 metadata, one device) and raises PATTN_ERR_INVALID_ARG before calling the library."""
    w = Workload("val", ((0, 20), (100, 1)), 32, 8, 128, 16, "bf16")
    db = DeviceBatch(generate(w, seed=4))
    args = lambda **kw: dict(dict(q=db.q, k_cache=db.k, v_cache=db.v, block_table=db.bt, cu_seqlens_q=db.cu,
                                  seq_lens=db.sl, scale=w.scale, num_kv_heads=8, block_size=16), **kw)
    bad = [
        dict(v_cache=db.v[:, :, :4]),
        dict(out=torch.empty_like(db.q, dtype=torch.float32)),
        dict(out=torch.empty((db.q.shape[0] + 1,) + tuple(db.q.shape[1:]), dtype=db.q.dtype, device="cuda")),
        dict(cu_seqlens_q=db.cu.long()),
        dict(seq_lens=db.sl.cpu()),
        dict(k_cache=db.k.float(), v_cache=db.v.float()),
    ]
    for kw in bad:
        with pytest.raises(P.PattnError) as ei:
            P.unified_attention(**args(**kw))
        assert ei.value.code == 1, kw.keys()


def test_default_workspace_is_per_stream():
    """Two calls on different streams without explicit workspaces get different cached buffers."""
    w = Workload("ws", ((0, 64), (900, 1), (1200, 1)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=5, dist="peaked")
    db = DeviceBatch(batch)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1, o2 = torch.empty_like(db.q), torch.empty_like(db.q)
    for _ in range(3):
        db.run(out=o1, stream=s1)
        db.run(out=o2, stream=s2)
    torch.cuda.synchronize()
    keys = [k for k in P._ws.buf if k[1] in (s1.cuda_stream, s2.cuda_stream)]
    assert len(keys) == 2
    assert torch.equal(o1, o2)
    assert_close(out_f64(o1), O.batch_attention(batch), "bf16", "per-stream workspace")


@pytest.mark.parametrize("case", [0, 4, 5, 6, 7, 8])
def test_baseline_kernel_parity(case):
    """The paper's baseline kernel (App. A, PATTN_FLAG_BASELINE: one warp per (token, head),
    tile = BLOCK_SIZE) against the oracle, bf16 and fp32, NHD / HND, block sizes 16, 80, 7, 5."""
    heads, D, bs, dt, layout, dist = CASES[case]
    rng = np.random.default_rng(77 + case)
    w = random_workload(rng, heads, D, bs, dt, max_seqs=5, max_len=400, decode_share=0.5)
    batch = generate(w, seed=case, dist=dist, layout=layout)
    db = DeviceBatch(batch)
    p = P.make_problem(db.q, db.k, w.num_kv_heads, w.block_size, db.bt, w.num_seqs, None, layout,
                       flags=P.FLAG_BASELINE)
    assert P.planned_kernels(p) == (1 << P.KERNEL_METADATA) | (1 << P.KERNEL_BASELINE)
    _check(batch, P.FLAG_BASELINE, f"baseline case {case} {w.seqs}")


def test_baseline_kernel_config1_fp32():
    _check(generate(CONFIGS["c1_tiny"], seed=1001), P.FLAG_BASELINE, "baseline c1")


# ---------------------------------------------------------------- CUDA-graph buckets (NEXT-1)
@pytest.mark.parametrize("two_streams", [False, True])
def test_graph_bucket_replays_with_fewer_sequences(two_streams):
    """Graphs recorded once per batch-size bucket (§6.2) and replayed for
    batches smaller than the bucket: padding sequences have q_b = 0, L_b = 0.  Decode-only
    buckets and a mixed bucket (prefill + decode, two streams), against the oracle."""
    from paper_2511_11581_b200.graphs import GraphBuckets

    # one KV cache holding every sequence the batches below use
    seqs = ((3000, 1), (100, 1), (4096, 1), (17, 1), (900, 1), (2500, 1), (0, 1))
    w = Workload("graphdec", seqs, 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=41, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    gb = GraphBuckets(db.k, db.v, 32, 8, 16, w.scale, buckets=(4, 8), max_query_len=1, max_seq_len=4097,
                      two_streams=two_streams)
    ref = O.batch_attention(batch)
    for ids in ([0, 1, 2, 3, 4], [5, 6, 1], [2]):  # bucket 8, bucket 4, bucket 4
        ids = np.array(ids)
        q = db.q[torch.from_numpy(ids).cuda()]
        bt = db.bt[torch.from_numpy(ids).cuda()]
        sl = db.sl[torch.from_numpy(ids).cuda()]
        cu = torch.arange(len(ids) + 1, dtype=torch.int32, device="cuda")
        out = gb.run(q, bt, cu, sl).clone()
        torch.cuda.synchronize()
        assert_close(out_f64(out), ref[ids], "bf16", f"graph bucket ids={ids.tolist()}")
        again = gb.run(q, bt, cu, sl)
        torch.cuda.synchronize()
        assert torch.equal(again, out)
    gb.close()

    # mixed bucket: up to 8 sequences, 400 query tokens (prefills + decodes), two streams
    w = Workload("graphmix", ((0, 200), (3000, 1), (64, 100), (900, 1), (1500, 1)), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=42, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    gb = GraphBuckets(db.k, db.v, 32, 8, 16, w.scale, buckets=(8,), max_query_len=256, max_seq_len=3001,
                      token_capacity={8: 400}, two_streams=two_streams)
    out = gb.run(db.q, db.bt, db.cu, db.sl).clone()
    torch.cuda.synchronize()
    assert_close(out_f64(out), O.batch_attention(batch), "bf16", "graph mixed bucket")
    gb.close()


# ---------------------------------------------------------------- error level (tighter than the tolerance)
@pytest.mark.parametrize("dist", ["uniform", "peaked"])
@pytest.mark.parametrize("heads,D", [((32, 8), 128), ((64, 8), 128), ((32, 8), 64)])
def test_bf16_error_stays_at_the_rounding_level(dist, heads, D):
    """The north_star tolerance (1e-2 abs + 1e-2 rel) is loose for small outputs; this checks the
    error against what the bf16 arithmetic allows (reading R12): P rounded to bf16 (relative
    2^-8 per element, so at most 2^-8 * max|v| on the weighted mean) plus the output cast (2^-8
    |out|), i.e. |err| <= 2^-8 (max|v| + |ref|) per element -- asserted with a 2x margin -- and
    the RMS error, where independent rounding errors average out, below 2^-9 * max|v|.  Every
    kernel path of the mixed batch (K1 prefill, K2 split decode + K3, short decodes)."""
    rng = np.random.default_rng(7 + D + heads[0])
    w = random_workload(rng, heads, D, 16, "bf16", max_seqs=8, max_len=3000, decode_share=0.5)
    batch = generate(w, seed=3, dist=dist, poison=True)
    ref = O.batch_attention(batch)
    gpu = out_f64(DeviceBatch(batch).run())
    vmax = float(np.abs(O.widen(batch.v_cache)[np.isfinite(O.widen(batch.v_cache))]).max())
    err = np.abs(gpu - ref)
    bound = 2.0 * 2.0 ** -8 * (vmax + np.abs(ref))
    assert (err <= bound).all(), f"{dist} {heads} D{D}: max err/bound {float((err / bound).max()):.2f}"
    rms = float(np.sqrt((err ** 2).mean()))
    assert rms <= 2.0 ** -9 * vmax, f"{dist} {heads} D{D}: rms err {rms:.2e}"


def test_two_stream_partition_follows_the_mix():
    """K5's SM partition (workspace header word kHdrPrefillCtas, the K1 share P) on batches of
    the same heads with a growing prefill share: P stays inside [1, #SMs - 1], grows with the
    prefill work, and the prefill-only / decode-heavy extremes land near the ends."""
    from paper_2511_11581_b200 import pattn

    num_sms = torch.cuda.get_device_properties(0).multi_processor_count
    shares = []
    for npre in (1, 2, 4, 8, 16):
        w = Workload(f"part{npre}", tuple([(0, 1024)] * npre + [(4096, 1)] * 48), 32, 8, 128, 16, "bf16")
        batch = generate(w, seed=npre, poison=False)
        db = DeviceBatch(batch)
        ws = torch.empty(1 << 24, dtype=torch.uint8, device="cuda")
        db.run(stream2=torch.cuda.Stream(), workspace=ws)
        P = pattn.workspace_prefill_sms(ws)
        assert 1 <= P <= num_sms - 1, (npre, P)
        shares.append(P)
    assert shares == sorted(shares), shares  # more prefill work -> more SMs for K1
    assert shares[-1] > shares[0]


# ---------------------------------------------------------------- shape fuzz
FUZZ_HEADS = [(32, 8), (64, 8), (28, 4), (48, 8), (16, 1), (8, 8), (40, 8), (12, 2), (96, 8), (24, 3)]


@pytest.mark.parametrize("i", range(48))
def test_shape_fuzz(i):
    """Seeded random shapes across every routing decision: heads (G = 1..12), head_dim 64/128,
    block sizes that K1/K2 take (16·k) and that only K4 takes (5, 7, 24), NHD/HND, bf16/fp32,
    ragged mixed batches with chunked prefills and long decodes, poisoned unused slots."""
    rng = np.random.default_rng(9000 + i)
    heads = FUZZ_HEADS[int(rng.integers(len(FUZZ_HEADS)))]
    D = int(rng.choice([64, 128]))
    bs = int(rng.choice([16, 32, 48, 80, 128, 5, 7, 24]))
    u = rng.random()
    dt = "f32" if u < 0.2 else ("f16" if u < 0.4 else "bf16")
    layout = "HND" if rng.random() < 0.4 else "NHD"
    w = random_workload(rng, heads, D, bs, dt, max_seqs=7, max_len=int(rng.choice([300, 1200, 2500])),
                        decode_share=float(rng.uniform(0.2, 0.8)))
    batch = generate(w, seed=i, dist="peaked", layout=layout, poison=True)
    _check(batch, 0, f"fuzz {i}: heads {heads} D{D} bs{bs} {dt} {layout} {w.seqs}")


# ---------------------------------------------------------------- decode kernels K2 and K2W
# K2W (head-wide TMA boxes, HB KV heads per item) is the default decode kernel when G <= 16 and
# 2 | Hkv; K2 (one KV head per item) stays for the rest and under PATTN_DECODE_WIDE=0.  Both are
# checked against the oracle on the same batches, for every HB K2W instantiates (PATTN_DECODE_WIDE_HB
# caps it), and the plan is checked to route where it says.
DECODE_CASES = [
    # heads, D, bs, dtype, layout
    ((32, 8), 128, 16, "bf16", "NHD"),
    ((64, 8), 128, 32, "bf16", "HND"),
    ((28, 4), 128, 16, "bf16", "NHD"),   # G = 7
    ((16, 2), 64, 48, "bf16", "NHD"),    # G = 8, D = 64, HB = 2
    ((32, 8), 64, 16, "f16", "HND"),
    ((12, 6), 128, 16, "bf16", "NHD"),   # Hkv = 6 -> HB = 2
    ((96, 8), 128, 16, "bf16", "HND"),   # G = 12: two head groups per KV head (8 + 4)
    ((64, 4), 64, 32, "f16", "NHD"),     # G = 16: two full head groups, D = 64
    ((40, 2), 128, 16, "bf16", "NHD"),   # G = 20 > 16: K2 in every case
]


@pytest.mark.parametrize("case", range(len(DECODE_CASES)))
@pytest.mark.parametrize("hb_cap", [8, 4, 2, 0])
def test_decode_wide_and_narrow(case, hb_cap, monkeypatch):
    heads, D, bs, dt, layout = DECODE_CASES[case]
    rng = np.random.default_rng(700 + case)
    seqs = [(int(rng.integers(1, 6000)), 1) for _ in range(9)] + [(int(rng.integers(0, 300)), int(rng.integers(2, 40)))]
    w = Workload(f"dec{case}", tuple(seqs), heads[0], heads[1], D, bs, dt)
    batch = generate(w, seed=case, dist="peaked", layout=layout, poison=True)
    if hb_cap == 0:
        monkeypatch.setenv("PATTN_DECODE_WIDE", "0")
    else:
        monkeypatch.setenv("PATTN_DECODE_WIDE_HB", str(hb_cap))
    db = DeviceBatch(batch)
    prob = P.make_problem(db.q, db.k, w.num_kv_heads, w.block_size, db.bt, w.num_seqs, kv_layout=layout)
    wide = bool(P.planned_kernels(prob) & P.PLAN_DECODE_WIDE)
    assert wide == (hb_cap > 0 and heads[0] // heads[1] <= 16), (heads, hb_cap, wide)
    ref = O.batch_attention(batch)
    for flags in (0, P.FLAG_FORCE_SPLIT, P.FLAG_NO_SPLIT):
        assert_close(out_f64(db.run(flags=flags)), ref, dt, f"{w.name} hb<={hb_cap} flags={flags}")


def test_decode_wide_equals_narrow_needles(monkeypatch):
    """Needle rows through both decode kernels: bit-exact V rows (one dominant key per KV head)."""
    w = Workload("wneedle", tuple([(3000 + 7 * i, 1) for i in range(6)]), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=77, dist="needle")
    v = O.widen(batch.v_cache)
    outs = []
    for wide in ("1", "0"):
        monkeypatch.setenv("PATTN_DECODE_WIDE", wide)
        out = DeviceBatch(batch).run(flags=P.FLAG_FORCE_SPLIT).cpu()
        for b in range(w.num_seqs):
            s = int(batch.cu_seqlens_q[b])
            for g in range(w.num_kv_heads):
                t = int(batch.needle_pos[b, g])
                row = torch.from_numpy(v[batch.block_table[b, t // 16], t % 16, g]).to(torch.bfloat16)
                for h in range(g * 4, g * 4 + 4):
                    assert torch.equal(out[s, h], row), (wide, b, g, h, t)
        outs.append(out)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("heads,D,bs,dt,layout", [((32, 8), 128, 7, "bf16", "NHD"), ((64, 8), 128, 24, "bf16", "HND"),
                                                  ((16, 2), 64, 5, "f16", "NHD"), ((28, 4), 128, 40, "bf16", "HND")])
@pytest.mark.parametrize("flags", [0, 0x4])
def test_gathered_decode_for_any_block_size(heads, D, bs, dt, layout, flags):
    """Block sizes that are not a multiple of 16: K2W gathers its ring entries row by row with
    cp.async (one block-table lookup per key, 16 keys spanning pages) -- planned as the decode
    kernel, split into segments that end inside pages, merged by K3, matching the oracle."""
    w = Workload("gather", ((20000, 1), (0, 70), (3000, 1), (17, 1), (700, 40), (9000, 1), (1, 1)), heads[0], heads[1],
                 D, bs, dt)
    batch = generate(w, seed=23 + bs, dist="peaked", poison=True, layout=layout)
    db = DeviceBatch(batch)
    p = P.make_problem(db.q, db.k, w.num_kv_heads, w.block_size, db.bt, w.num_seqs, None, layout, 70, 20001, flags)
    assert P.planned_kernels(p) & (1 << P.KERNEL_DECODE) and P.planned_kernels(p) & P.PLAN_DECODE_WIDE
    a = db.run(flags=flags).clone()
    assert_close(out_f64(a), O.batch_attention(batch), dt, f"gathered K2W {heads} D{D} bs={bs} flags={flags}")
    assert torch.equal(db.run(flags=flags), a)


def test_gathered_decode_needles():
    """Needle rows through the gathered K2W at bs 7: bit-exact V rows (paging arithmetic)."""
    w = Workload("gneedle", tuple([(2999 + 5 * i, 1) for i in range(5)]), 32, 8, 128, 7, "bf16")
    batch = generate(w, seed=71, dist="needle")
    out = DeviceBatch(batch).run(flags=P.FLAG_FORCE_SPLIT).cpu()
    v = O.widen(batch.v_cache)
    for b in range(w.num_seqs):
        s = int(batch.cu_seqlens_q[b])
        for g in range(w.num_kv_heads):
            t = int(batch.needle_pos[b, g])
            row = torch.from_numpy(v[batch.block_table[b, t // 7], t % 7, g]).to(torch.bfloat16)
            for h in range(g * 4, g * 4 + 4):
                assert torch.equal(out[s, h], row), (b, g, h, t)


@pytest.mark.parametrize("heads,D,bs,dt,layout", [((32, 8), 128, 7, "bf16", "NHD"), ((64, 8), 128, 24, "bf16", "HND"),
                                                  ((8, 8), 64, 5, "f16", "NHD"), ((28, 4), 128, 40, "bf16", "HND"),
                                                  ((96, 8), 128, 12, "bf16", "NHD")])
def test_gathered_prefill_for_any_block_size(heads, D, bs, dt, layout):
    """Block sizes that are not a multiple of 16 on the tensor-core prefill: K1's producers gather
    each 64-key tile row by row with cp.async (keys past the visible range zero-filled) --
    planned, matching the oracle on prefills with and without context, ragged tails."""
    w = Workload("gpre", ((0, 333), (500, 130), (3, 1), (61, 200), (1000, 1), (0, 17)), heads[0], heads[1], D, bs, dt)
    batch = generate(w, seed=31 + bs, dist="peaked", poison=True, layout=layout)
    db = DeviceBatch(batch)
    p = P.make_problem(db.q, db.k, w.num_kv_heads, w.block_size, db.bt, w.num_seqs, None, layout, 333, 1000)
    assert P.planned_kernels(p) & (1 << P.KERNEL_PREFILL)
    a = db.run().clone()
    assert_close(out_f64(a), O.batch_attention(batch), dt, f"gathered K1 {heads} D{D} bs={bs}")
    assert torch.equal(db.run(), a)



def test_large_batch_multi_pass_metadata():
    """More sequences than K5's 1024 threads (its multi-pass scan), decodes on K2W and K3,
    prefills on K1, empty sequences in between: plan bit-exact vs the oracle's metadata and the
    output vs the oracle."""
    rng = np.random.default_rng(1500)
    seqs = []
    for i in range(1500):
        u = rng.random()
        if u < 0.9:
            seqs.append((int(rng.integers(1, 700)), 1))
        elif u < 0.97:
            seqs.append((int(rng.integers(0, 200)), int(rng.integers(2, 90))))
        else:
            seqs.append((0, 0))
    w = Workload("bigB", tuple(seqs), 32, 8, 128, 16, "bf16")
    batch = generate(w, seed=1500, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    prob = P.make_problem(db.q, db.k, w.num_kv_heads, w.block_size, db.bt, w.num_seqs)
    plan = P.debug_plan(prob, db.cu, db.sl).cpu().numpy()
    B = w.num_seqs
    qlens = np.diff(batch.cu_seqlens_q)
    dec = qlens == 1
    cu_qb_ref = M.build_batch_meta(np.concatenate([[0], np.cumsum(np.where(dec, 0, qlens))]),
                                   np.where(dec, 0, batch.seq_lens), int(plan[3]))["cu_q_blocks"]
    assert plan[8:8 + B + 1].tolist() == cu_qb_ref.tolist()
    assert plan[1] == int(dec.sum())
    _check(batch, 0, "1500 sequences")


K2W_MATRIX = [
    # heads (Hq, Hkv), D, bs, dtype, layout -- G = 1 .. 16, TMA and gathered entries, NHD / HND
    ((8, 8), 128, 32, "bf16", "HND"),    # G 1, HB 8
    ((16, 8), 64, 64, "f16", "NHD"),     # G 2
    ((16, 4), 128, 128, "bf16", "HND"),  # G 4, HB 4, bs 128
    ((64, 8), 128, 9, "bf16", "NHD"),    # G 8, gathered (bs 9)
    ((48, 4), 64, 16, "bf16", "HND"),    # G 12, HB 4, two head groups
    ((32, 2), 128, 33, "f16", "HND"),    # G 16, HB 2, gathered (bs 33)
]


@pytest.mark.parametrize("case", range(len(K2W_MATRIX)))
def test_k2w_matrix(case):
    """K2W across GQA ratios 1..16 (one or two head groups per KV head), heads per box 2/4/8,
    TMA boxes and cp.async-gathered entries, both layouts: planned as K2W, split and unsplit
    decodes next to a prefill, matching the oracle; needles bit-exact on the same shapes."""
    heads, D, bs, dt, layout = K2W_MATRIX[case]
    w = Workload(f"k2wm{case}", ((5000, 1), (130, 1), (2, 1), (0, 77), (12000, 1), (700, 1)), heads[0], heads[1], D,
                 bs, dt)
    batch = generate(w, seed=900 + case, dist="peaked", poison=True, layout=layout)
    db = DeviceBatch(batch)
    p = P.make_problem(db.q, db.k, w.num_kv_heads, w.block_size, db.bt, w.num_seqs, None, layout, 77, 12001)
    assert P.planned_kernels(p) & P.PLAN_DECODE_WIDE
    ref = O.batch_attention(batch)
    for flags in (0, P.FLAG_FORCE_SPLIT):
        assert_close(out_f64(db.run(flags=flags)), ref, dt, f"{w.name} flags={flags}")
    if dt == "bf16":
        wn = Workload(f"k2wn{case}", ((3000, 1), (411, 1)), heads[0], heads[1], D, bs, dt)
        nb = generate(wn, seed=950 + case, dist="needle", layout=layout)
        out = DeviceBatch(nb).run(flags=P.FLAG_FORCE_SPLIT).cpu()
        v = O.widen(nb.v_cache)
        G = heads[0] // heads[1]
        for b in range(wn.num_seqs):
            s = int(nb.cu_seqlens_q[b])
            for g in range(wn.num_kv_heads):
                t = int(nb.needle_pos[b, g])
                blk, slot = int(nb.block_table[b, t // bs]), t % bs
                row = v[blk, g, slot] if layout == "HND" else v[blk, slot, g]
                row = torch.from_numpy(row).to(torch.bfloat16)
                for h in range(g * G, (g + 1) * G):
                    assert torch.equal(out[s, h], row), (case, b, g, h, t)


@pytest.mark.parametrize("G,D", [(4, 128), (8, 128), (4, 64)])
def test_prefill_claim_groups(G, D, monkeypatch):
    """Batches whose prefills all have the same number of Q blocks: K1 claims rank by rank within
    groups of sequences (K5: kHdrQbUniform / kHdrQbGroup).  Every group size -- one sequence, a
    short last group, all sequences -- must cover every item: oracle parity, and bitwise equal
    outputs across group sizes (the order moves items between CTAs, not their arithmetic)."""
    seqs = ((1000, 300), (7, 1), (0, 300), (2500, 300), (3000, 1), (333, 300), (64, 300))
    w = Workload("claim_groups", seqs, 8 * G, 8, D, 16, "bf16")
    batch = generate(w, seed=71 + G + D, dist="peaked", poison=True)
    db = DeviceBatch(batch)
    outs = []
    for mb in ("1", "11", "16", "100000"):  # ~5 MB of K/V per sequence: groups of 1, 2, 3, 5
        monkeypatch.setenv("PATTN_K1_GROUP_MB", mb)
        outs.append(db.run().clone())
        if mb == "11":
            assert_close(out_f64(outs[-1]), O.batch_attention(batch), batch.dtype, f"claim groups G={G} D={D}")
    s2 = torch.cuda.Stream()
    outs.append(db.run(stream2=s2).clone())  # two-stream partition, group of 5 (env 100000)
    for o in outs[1:]:
        assert torch.equal(outs[0], o)


@pytest.mark.parametrize("hq", [32, 64, 48])  # G = 4, 8, 6: BLOCK_Q 64 and 32 (closed form), 42 (walk)
def test_partition_model_tile_count(hq, monkeypatch):
    """K5's SM split from its cost model (k5_metadata.cu): the K1 work term counts (Q block,
    128-key tile) pairs with a closed form over one period of the ceilings when BLOCK_Q is a
    power of two.  Recomputed here by walking every Q block (float32 like the kernel; +-1 SM for
    FMA contraction), on ragged contexts and Q lengths that are not multiples of BLOCK_Q."""
    from paper_2511_11581_b200 import pattn

    monkeypatch.setenv("PATTN_K1_TILE_US", "2.2")
    monkeypatch.setenv("PATTN_K2W_SM_GBS", "10")  # low decode rate, no HBM cap: the split lands mid-range,
    monkeypatch.setenv("PATTN_HBM_GBS", "100000")  # where it moves ~S/4 SMs per unit of relative K1 work
    S = torch.cuda.get_device_properties(0).multi_processor_count
    rng = np.random.default_rng(hq)
    for rep in range(4):
        pre = [(int(rng.integers(0, 3000)), int(rng.integers(2, 1500))) for _ in range(int(rng.integers(2, 7)))]
        dec = [(int(rng.integers(1000, 6000)), 1) for _ in range(int(rng.integers(8, 30)))]
        w = Workload(f"pm{hq}_{rep}", tuple(pre + dec), hq, 8, 128, 16, "bf16")
        db = DeviceBatch(generate(w, seed=rep, poison=False))
        ws = torch.zeros(1 << 24, dtype=torch.uint8, device="cuda")
        db.run(stream2=torch.cuda.Stream(), workspace=ws)
        bq = int(ws[12:16].view(torch.int32).item())
        tiles = sum(-(-(c + min(t0 + bq, q)) // 128) for c, q in pre for t0 in range(0, q, bq))
        keys = sum(c + 1 for c, _ in dec)
        f = np.float32
        tp = f(tiles) * f(8) * f(2.2) * f(1e-6)
        b = f(10) * f(1e9)
        nbytes = f(keys) * f(8) * f(128) * f(4)
        cstar = f(S) * tp * b / (tp * b + nbytes)
        chbm = f(S) - f(100000) / f(10)
        want = max(1, min(int(max(cstar, chbm) + f(0.5)), S - 1))
        got = pattn.workspace_prefill_sms(ws)
        assert abs(got - want) <= 1, (hq, rep, bq, tiles, got, want)
        assert S // 8 < want < S - S // 8, (hq, rep, want)  # mid-range: sensitive to the tile count
