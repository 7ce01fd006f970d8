"""fp64 paged causal attention oracle (ctypes wrapper over oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definition followed (pattn_oracle.c header): Eq. 1 and Eq. 2 (§4.1,
P:212-216), terminology context/query/sequence/prefix length (§4.2,
P:304-317), all K/V read from the paged cache through the block table (App. A
P:10-14, §4.3), contiguous GQA grouping (§4.1).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile pattn_oracle.c (gcc -O2 -fopenmp, no -ffast-math: plain IEEE fp64)."""
    src = os.path.join(_HERE, "pattn_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _LIB_PATH, src, "-lm"]
        )
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i32p = ctypes.POINTER(ctypes.c_int32)
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        I, L = ctypes.c_int, ctypes.c_int64
        lib.oracle_paged_attention.restype = ctypes.c_int
        lib.oracle_paged_attention.argtypes = [
            I, i32p, i32p, I, I, I, I, f32p, L, L, f32p, f32p, L, L, L, i32p, L,
            ctypes.c_double, i64p, L, f64p, I,
        ]
        lib.oracle_validate.restype = ctypes.c_int
        lib.oracle_validate.argtypes = [I, i32p, i32p, I, I, i32p, L, I]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def widen(a: np.ndarray) -> np.ndarray:
    """Storage -> fp32, exactly: bf16 bit patterns (uint16) are shifted into the fp32 high half."""
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32)
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def validate(cu_seqlens_q, seq_lens, block_size, num_blocks, block_table) -> int:
    lib = _load()
    cu = np.ascontiguousarray(cu_seqlens_q, np.int32)
    sl = np.ascontiguousarray(seq_lens, np.int32)
    bt = np.ascontiguousarray(block_table, np.int32)
    return int(lib.oracle_validate(len(sl), _ptr(cu, ctypes.c_int32), _ptr(sl, ctypes.c_int32), block_size,
                                   num_blocks, _ptr(bt, ctypes.c_int32), bt.shape[1], bt.shape[1]))


def paged_attention(
    q: np.ndarray,
    k_cache: np.ndarray,
    v_cache: np.ndarray,
    block_table: np.ndarray,
    cu_seqlens_q: np.ndarray,
    seq_lens: np.ndarray,
    scale: float,
    num_kv_heads: int,
    block_size: int,
    layout: str = "NHD",
    rows: Optional[Sequence[int]] = None,
    threads: int = 0,
) -> np.ndarray:
    """Attention output in fp64.

    q: [T, Hq, D]; k_cache/v_cache: [num_blocks, bs, Hkv, D] ("NHD") or
    [num_blocks, Hkv, bs, D] ("HND"), fp32 or bf16 bits (uint16).
    rows: optional flat row ids (tok*Hq + h); returns [len(rows), D] then, else [T, Hq, D].
    """
    lib = _load()
    qf = widen(q)
    kf = widen(k_cache)
    vf = widen(v_cache)
    T, Hq, D = qf.shape
    bt = np.ascontiguousarray(block_table, np.int32)
    cu = np.ascontiguousarray(cu_seqlens_q, np.int32)
    sl = np.ascontiguousarray(seq_lens, np.int32)
    B = len(sl)
    if layout == "NHD":
        nb, bs, hkv, d = kf.shape
        strides = (bs * hkv * d, hkv * d, d)
    else:
        nb, hkv, bs, d = kf.shape
        strides = (hkv * bs * d, d, bs * d)
    assert bs == block_size and hkv == num_kv_heads and d == D
    if rows is None:
        rr = None
        n = T * Hq
    else:
        rr = np.ascontiguousarray(rows, np.int64)
        n = len(rr)
    out = np.empty((n, D), dtype=np.float64)
    err = lib.oracle_paged_attention(
        B, _ptr(cu, ctypes.c_int32), _ptr(sl, ctypes.c_int32), Hq, num_kv_heads, D, block_size,
        _ptr(qf, ctypes.c_float), Hq * D, D,
        _ptr(kf, ctypes.c_float), _ptr(vf, ctypes.c_float), strides[0], strides[1], strides[2],
        _ptr(bt, ctypes.c_int32), bt.shape[1], float(scale),
        None if rr is None else _ptr(rr, ctypes.c_int64), n,
        _ptr(out, ctypes.c_double), int(threads),
    )
    if err:
        raise ValueError(f"oracle_paged_attention error {err}")
    return out if rows is not None else out.reshape(T, Hq, D)


def batch_attention(batch, rows=None, threads: int = 0) -> np.ndarray:
    """Convenience: run on a workloads.Batch."""
    w = batch.workload
    return paged_attention(batch.q, batch.k_cache, batch.v_cache, batch.block_table, batch.cu_seqlens_q,
                           batch.seq_lens, w.scale, w.num_kv_heads, w.block_size, layout=batch.layout,
                           rows=rows, threads=threads)
