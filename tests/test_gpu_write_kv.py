"""GPU parity of the paged KV write (pattn_write_kv, K6) against oracle/kvcache.py: the
whole caches must be BIT-EXACT (it is a copy; untouched rows keep their NaN poison), for
bf16 and fp32, NHD and HND layouts, block sizes 16 / 32 / 80, ragged mixed batches, an
empty batch and the config-3 shape.  Then write -> attend through both libpattn calls
against the oracle."""
import numpy as np
import pytest
import torch

from oracle import attention as O
from oracle import kvcache as KV
from workloads import CONFIGS, Workload, generate
from workloads.gen import _uniform

from gpu_helpers import DeviceBatch, assert_close, out_f64, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _bits(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy().view(np.uint32)


def _run(w, layout, seed):
    from paper_2511_11581_b200 import pattn

    b = generate(w, seed=seed, layout="NHD")
    rng = np.random.Generator(np.random.PCG64(seed + 1))
    T, hkv, d = w.num_tokens, w.num_kv_heads, w.head_dim
    k_new = _uniform(rng, (T, hkv, d), w.dtype)
    v_new = _uniform(rng, (T, hkv, d), w.dtype)
    ref_k, ref_v = KV.write_kv(k_new, v_new, b.k_cache, b.v_cache, b.block_table, b.cu_seqlens_q, b.seq_lens,
                               w.block_size)
    kc, vc = b.k_cache, b.v_cache
    if layout == "HND":
        kc, vc = kc.transpose(0, 2, 1, 3), vc.transpose(0, 2, 1, 3)
    kc, vc = to_torch(np.ascontiguousarray(kc)), to_torch(np.ascontiguousarray(vc))
    pattn.write_kv(to_torch(k_new), to_torch(v_new), kc, vc, torch.from_numpy(b.block_table).cuda(),
                   torch.from_numpy(b.cu_seqlens_q).cuda(), torch.from_numpy(b.seq_lens).cuda(), w.block_size,
                   kv_layout=layout)
    torch.cuda.synchronize()
    if layout == "HND":
        kc, vc = kc.transpose(1, 2), vc.transpose(1, 2)
    gk, gv = _bits(kc.contiguous()), _bits(vc.contiguous())
    view = np.uint16 if w.dtype == "bf16" else np.uint32
    assert np.array_equal(gk, ref_k.view(view)), "K cache differs from the oracle"
    assert np.array_equal(gv, ref_v.view(view)), "V cache differs from the oracle"
    return b, k_new, v_new, ref_k, ref_v


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("layout", ["NHD", "HND"])
@pytest.mark.parametrize("bs", [16, 32, 80])
def test_write_kv_bit_exact(dtype, layout, bs):
    seqs = ((0, 70), (3000, 1), (100, 1), (33, 17), (0, 1), (5, 0), (79, 161))
    _run(Workload("kvw", seqs, 32, 8, 128, bs, dtype), layout, seed=77 + bs)


def test_write_kv_d64_single_head_many_seqs():
    seqs = tuple((int(c), int(q)) for c, q in zip(np.arange(300) * 7 % 500, np.arange(300) % 5))
    _run(Workload("kvw_many", seqs, 8, 1, 64, 16, "bf16"), "NHD", seed=5)


def test_write_kv_empty_batch_is_noop():
    _run(Workload("kvw_empty", ((10, 0), (3, 0)), 8, 2, 128, 16, "bf16"), "NHD", seed=6)


def test_write_kv_config3_shape():
    _run(CONFIGS["c3_mixed8b"], "NHD", seed=3)


def test_write_then_attend():
    # fill the query tokens' K/V with write_kv, then attend: equals the oracle on the oracle's cache
    w = Workload("kvw_attn", ((0, 130), (2000, 1), (64, 40), (777, 1)), 32, 8, 128, 16, "bf16")
    b, k_new, v_new, ref_k, ref_v = _run(w, "NHD", seed=8)
    b.k_cache, b.v_cache = ref_k, ref_v
    db = DeviceBatch(b)
    from paper_2511_11581_b200 import pattn

    db.k.fill_(float("nan"))
    db.v.fill_(float("nan"))
    # the device cache gets the old rows from the generator plus the written ones
    old = generate(w, seed=8)
    db.k.copy_(to_torch(old.k_cache))
    db.v.copy_(to_torch(old.v_cache))
    pattn.write_kv(to_torch(k_new), to_torch(v_new), db.k, db.v, db.bt, db.cu, db.sl, w.block_size)
    gpu = out_f64(db.run())
    assert_close(gpu, O.batch_attention(b), "bf16", "write_kv -> unified_attention")
