"""CPU-only checks of the C-ABI boundary: libpattn.so loads without a GPU, exports every
symbol include/pattn.h declares, and its host-only entry points (status strings, host
metadata validation, workspace sizing, planned launch count) behave as documented.
No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "pattn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"PATTN_API\s+[\w\s\*]+?\b(pattn_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2511_11581_b200 import pattn

    if not os.path.exists(pattn.LIB_PATH):
        import subprocess

        subprocess.check_call(["make", "-s", "-C", ROOT])
    return pattn


def test_header_declares_expected_api():
    fns = _header_functions()
    assert "pattn_unified_attention" in fns and len(fns) >= 10


def test_library_exports_every_header_symbol(lib):
    so = lib.load()
    for name in _header_functions():
        assert hasattr(so, name), f"libpattn.so does not export {name}"
    assert set(_header_functions()) == set(lib.EXPORTS)


def test_status_strings_and_version(lib):
    so = lib.load()
    for code, name in lib.STATUS.items():
        assert so.pattn_status_string(code).decode() == name
    assert lib.version() >= 100


def _problem(lib, B=2, T=17, Hq=4, Hkv=1, D=64, bs=16, nb=4, maxb=3, dtype=0, flags=0):
    p = lib.Problem()
    p.num_seqs, p.num_tokens, p.num_q_heads, p.num_kv_heads, p.head_dim = B, T, Hq, Hkv, D
    p.block_size, p.num_blocks, p.max_blocks_per_seq, p.dtype, p.flags = bs, nb, maxb, dtype, flags
    p.q_stride_tok, p.q_stride_head = Hq * D, D
    p.kv_stride_blk, p.kv_stride_tok, p.kv_stride_head = bs * Hkv * D, Hkv * D, D
    p.bt_stride = maxb
    p.o_stride_tok, p.o_stride_head = Hq * D, D
    return p


def test_validate_metadata_host_matches_oracle_codes(lib):
    from oracle import attention as O

    p = _problem(lib)
    cu = np.array([0, 16, 17], np.int32)
    sl = np.array([16, 33], np.int32)
    bt = np.array([[0, -1, -1], [1, 2, 3]], np.int32)
    assert lib.validate_metadata_host(p, cu, sl, bt) == 0 == O.validate(cu, sl, 16, 4, bt)
    bad_q = np.array([15, 33], np.int32)  # q_b > L_b
    assert lib.validate_metadata_host(p, cu, bad_q, bt) == 3 == O.validate(cu, bad_q, 16, 4, bt)
    bad_bt = np.array([[0, -1, -1], [1, 2, 4]], np.int32)  # block id 4 >= num_blocks
    assert lib.validate_metadata_host(p, cu, sl, bad_bt) == 4 == O.validate(cu, sl, 16, 4, bad_bt)
    long_sl = np.array([16, 49], np.int32)  # needs 4 blocks > max_blocks_per_seq
    assert lib.validate_metadata_host(p, cu, long_sl, bt) == 4
    p0 = _problem(lib, B=0)
    assert lib.validate_metadata_host(p0, cu, sl, bt) == 2
    assert lib.validate_metadata_host(p, np.array([1, 16, 17], np.int32), sl, bt) == 3


def test_workspace_and_planned_launches(lib, monkeypatch):
    so = lib.load()
    p = _problem(lib)  # fp32 -> metadata + generic (Q blocks + split decode segments) + reduce
    assert so.pattn_workspace_size(ctypes.byref(p)) > 0
    assert lib.planned_launches(p) == 3
    assert lib.planned_kernels(p) == (1 << lib.KERNEL_METADATA) | (1 << lib.KERNEL_GENERIC) | (
        1 << lib.KERNEL_REDUCE)
    pb = _problem(lib, Hq=32, Hkv=8, D=128, dtype=1, T=64, B=64, nb=16448, maxb=257)
    pb.max_query_len = 1
    assert lib.planned_launches(pb) == 3  # metadata + decode + reduce
    # G = 4, Hkv = 8: the decode kind runs as K2W (8 KV heads per TMA box)
    assert lib.planned_kernels(pb) == (1 << lib.KERNEL_METADATA) | (1 << lib.KERNEL_DECODE) | (
        1 << lib.KERNEL_REDUCE) | lib.PLAN_DECODE_WIDE
    monkeypatch.setenv("PATTN_DECODE_WIDE", "0")  # K2 (one KV head per item)
    assert lib.planned_kernels(pb) == (1 << lib.KERNEL_METADATA) | (1 << lib.KERNEL_DECODE) | (
        1 << lib.KERNEL_REDUCE)
    monkeypatch.delenv("PATTN_DECODE_WIDE")
    pg = _problem(lib, Hq=128, Hkv=4, D=128, dtype=1, T=64, B=64, nb=16448, maxb=257)  # G = 32: K2
    pg.max_query_len = 1
    assert not lib.planned_kernels(pg) & lib.PLAN_DECODE_WIDE
    pb.max_query_len = 2048
    assert lib.planned_launches(pb) == 4  # + the Q-block kernel
    pb.flags = lib.FLAG_FORCE_GENERIC
    assert lib.planned_launches(pb) == 3
    bad = _problem(lib, D=96)
    assert so.pattn_workspace_size(ctypes.byref(bad)) == 0
    assert so.pattn_hostio_workspace_size(ctypes.byref(p)) > so.pattn_workspace_size(ctypes.byref(p))
