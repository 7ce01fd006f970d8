"""Thin Python binding of libpattn (include/pattn.h) -- argument marshalling only.

Every step of the attention path runs inside libpattn's CUDA kernels; this module
only turns torch tensors into pointers, sizes and strides, keeps a cached device
workspace, and calls the C ABI through ctypes.  There is no CPU fallback: if the
shared library is missing, importing the call raises.

Names follow north_star: unified_attention(q, k_cache, v_cache, block_table,
cu_seqlens_q, seq_lens, scale, num_kv_heads, block_size, out).
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PATTN_LIB") or os.path.join(_HERE, "lib", "libpattn.so")  # PATTN_LIB: A/B builds

PATTN_OK = 0
STATUS = {
    0: "PATTN_OK",
    1: "PATTN_ERR_INVALID_ARG",
    2: "PATTN_ERR_EMPTY_BATCH",
    3: "PATTN_ERR_INVALID_SEQUENCE",
    4: "PATTN_ERR_INDEX_OUT_OF_RANGE",
    5: "PATTN_ERR_UNSUPPORTED",
    6: "PATTN_ERR_WORKSPACE_TOO_SMALL",
    7: "PATTN_ERR_CUDA",
}
DTYPE_F32, DTYPE_BF16, DTYPE_F16 = 0, 1, 2
FLAG_FORCE_GENERIC, FLAG_NO_SPLIT, FLAG_FORCE_SPLIT, FLAG_SERIAL, FLAG_BASELINE = 0x1, 0x2, 0x4, 0x8, 0x10
KERNEL_METADATA, KERNEL_PREFILL, KERNEL_DECODE, KERNEL_REDUCE, KERNEL_GENERIC, KERNEL_BASELINE, KERNEL_COUNT = range(7)
KERNEL_NAMES = ["metadata", "prefill", "decode", "reduce", "generic", "baseline"]
PLAN_DECODE_WIDE = 1 << 8  # planned_kernels(): the decode kind runs as K2W (head-wide TMA boxes)


class PattnError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {STATUS.get(code, code)}")
        self.code = code


class Problem(ctypes.Structure):
    _fields_ = [
        ("num_seqs", ctypes.c_int32),
        ("num_tokens", ctypes.c_int32),
        ("num_q_heads", ctypes.c_int32),
        ("num_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("block_size", ctypes.c_int32),
        ("num_blocks", ctypes.c_int32),
        ("max_blocks_per_seq", ctypes.c_int32),
        ("max_query_len", ctypes.c_int32),
        ("max_seq_len", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("q_stride_tok", ctypes.c_int64),
        ("q_stride_head", ctypes.c_int64),
        ("kv_stride_blk", ctypes.c_int64),
        ("kv_stride_tok", ctypes.c_int64),
        ("kv_stride_head", ctypes.c_int64),
        ("bt_stride", ctypes.c_int64),
        ("o_stride_tok", ctypes.c_int64),
        ("o_stride_head", ctypes.c_int64),
    ]


class ExecOpts(ctypes.Structure):
    _fields_ = [("stream2", ctypes.c_void_p), ("events", ctypes.c_void_p * (2 * KERNEL_COUNT))]


_lib = None
_lock = threading.Lock()

EXPORTS = [
    "pattn_workspace_size",
    "pattn_unified_attention",
    "pattn_unified_attention_ex",
    "pattn_hostio_workspace_size",
    "pattn_unified_attention_hostio",
    "pattn_status_string",
    "pattn_validate_metadata_host",
    "pattn_debug_plan",
    "pattn_planned_launches",
    "pattn_planned_kernels",
    "pattn_last_error",
    "pattn_version",
    "pattn_write_kv",
    "pattn_set_tuning_tree",
    "pattn_plan_tuning",
    "pattn_graph_capture",
    "pattn_graph_launch",
    "pattn_graph_destroy",
]


def load() -> ctypes.CDLL:
    """Load libpattn.so (fail loudly when it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"libpattn not built: {LIB_PATH} missing (run `make` or __graft_entry__.build())")
            lib = ctypes.CDLL(LIB_PATH)
            P = ctypes.POINTER(Problem)
            vp, i32p, sz = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.c_size_t
            lib.pattn_workspace_size.restype = sz
            lib.pattn_workspace_size.argtypes = [P]
            lib.pattn_hostio_workspace_size.restype = sz
            lib.pattn_hostio_workspace_size.argtypes = [P]
            common = [P, vp, vp, vp, vp, vp, vp, ctypes.c_float, vp, vp, sz, vp]
            lib.pattn_unified_attention.restype = ctypes.c_int
            lib.pattn_unified_attention.argtypes = common
            lib.pattn_unified_attention_ex.restype = ctypes.c_int
            lib.pattn_unified_attention_ex.argtypes = common + [ctypes.POINTER(ExecOpts)]
            lib.pattn_unified_attention_hostio.restype = ctypes.c_int
            lib.pattn_unified_attention_hostio.argtypes = common
            lib.pattn_status_string.restype = ctypes.c_char_p
            lib.pattn_status_string.argtypes = [ctypes.c_int]
            lib.pattn_validate_metadata_host.restype = ctypes.c_int
            lib.pattn_validate_metadata_host.argtypes = [P, i32p, i32p, i32p]
            lib.pattn_debug_plan.restype = ctypes.c_int
            lib.pattn_debug_plan.argtypes = [P, vp, vp, vp, ctypes.c_int32, vp, sz, vp]
            lib.pattn_planned_launches.restype = ctypes.c_int32
            lib.pattn_planned_launches.argtypes = [P]
            lib.pattn_planned_kernels.restype = ctypes.c_int32
            lib.pattn_planned_kernels.argtypes = [P]
            if hasattr(lib, "pattn_write_kv"):  # absent only in older A/B builds (PATTN_LIB)
                lib.pattn_write_kv.restype = ctypes.c_int
                lib.pattn_write_kv.argtypes = [P, vp, vp, ctypes.c_int64, ctypes.c_int64, vp, vp, vp, vp, vp, vp]
            if hasattr(lib, "pattn_set_tuning_tree"):  # absent only in older A/B builds
                lib.pattn_set_tuning_tree.restype = ctypes.c_int
                lib.pattn_set_tuning_tree.argtypes = [vp, ctypes.c_int32]
                lib.pattn_plan_tuning.restype = ctypes.c_int
                lib.pattn_plan_tuning.argtypes = [P, vp]
            if hasattr(lib, "pattn_graph_capture"):  # absent only in older A/B builds
                lib.pattn_graph_capture.restype = ctypes.c_int
                lib.pattn_graph_capture.argtypes = common + [vp, ctypes.POINTER(vp)]
                lib.pattn_graph_launch.restype = ctypes.c_int
                lib.pattn_graph_launch.argtypes = [vp, vp]
                lib.pattn_graph_destroy.restype = ctypes.c_int
                lib.pattn_graph_destroy.argtypes = [vp]
            lib.pattn_version.restype = ctypes.c_int32
            lib.pattn_last_error.restype = ctypes.c_char_p
            _lib = lib
            # the fitted planner heuristics (scripts/tune.py -> tuning_tree.json, §4.2)
            tree_path = os.path.join(_HERE, "tuning_tree.json")
            if hasattr(lib, "pattn_set_tuning_tree") and os.path.exists(tree_path) and \
                    not os.environ.get("PATTN_NO_TUNING_TREE"):
                import json

                from . import tuner

                nodes = tuner.flatten(json.load(open(tree_path)))
                arr = (tuner.TreeNode * len(nodes))(*nodes)
                code = lib.pattn_set_tuning_tree(arr, len(nodes))
                if code != PATTN_OK:
                    raise PattnError(code, f"pattn_set_tuning_tree({tree_path})")
    return _lib


def _check(code: int, where: str):
    if code != PATTN_OK:
        detail = load().pattn_last_error().decode() if code == 7 else ""
        raise PattnError(code, f"{where} {detail}".strip())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return DTYPE_F32
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    if t.dtype == torch.float16:
        return DTYPE_F16
    raise PattnError(5, f"dtype {t.dtype}")


def make_problem(
    q: torch.Tensor,
    k_cache: torch.Tensor,
    num_kv_heads: int,
    block_size: int,
    block_table: torch.Tensor,
    num_seqs: int,
    out: Optional[torch.Tensor] = None,
    kv_layout: str = "NHD",
    max_query_len: Optional[int] = None,
    max_seq_len: Optional[int] = None,
    flags: int = 0,
) -> Problem:
    """Sizes and element strides from tensor shapes (host-known; no device reads)."""
    T, Hq, D = q.shape
    if kv_layout == "NHD":
        nb, bs, hkv, d = k_cache.shape
        s_blk, s_tok, s_head, s_d = k_cache.stride()
    elif kv_layout == "HND":
        nb, hkv, bs, d = k_cache.shape
        s_blk, s_head, s_tok, s_d = k_cache.stride()
    else:
        raise ValueError(kv_layout)
    if bs != block_size or hkv != num_kv_heads or d != D or s_d != 1 or q.stride(2) != 1:
        raise PattnError(1, "shape/stride mismatch")
    o = out if out is not None else q
    p = Problem()
    p.num_seqs = num_seqs
    p.num_tokens = T
    p.num_q_heads = Hq
    p.num_kv_heads = num_kv_heads
    p.head_dim = D
    p.block_size = block_size
    p.num_blocks = nb
    p.max_blocks_per_seq = block_table.shape[1]
    p.max_query_len = int(max_query_len) if max_query_len is not None else 0
    p.max_seq_len = int(max_seq_len) if max_seq_len is not None else 0
    p.dtype = _dtype_code(q)
    p.flags = flags
    p.q_stride_tok, p.q_stride_head = q.stride(0), q.stride(1)
    p.kv_stride_blk, p.kv_stride_tok, p.kv_stride_head = s_blk, s_tok, s_head
    p.bt_stride = block_table.stride(0)
    p.o_stride_tok, p.o_stride_head = o.stride(0), o.stride(1)
    return p


class _Workspace:
    """Cached default workspaces, one per (device, stream): two calls on different streams
    never share one (the C ABI requires distinct workspaces for concurrent calls).  A buffer
    that is outgrown is retired but kept alive (never returned to the caching allocator), so
    kernels still in flight on any stream and CUDA graphs captured with it stay valid."""

    def __init__(self):
        self.buf = {}
        self.retired = []
        self.lock = threading.Lock()

    def get(self, nbytes: int, device: torch.device, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        dev = device.index if device.index is not None else torch.cuda.current_device()
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        key = (dev, int(s.cuda_stream))
        with self.lock:
            b = self.buf.get(key)
            if b is None or b.numel() < nbytes:
                if b is not None:
                    self.retired.append(b)
                b = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=torch.device("cuda", dev))
                self.buf[key] = b
            return b


_ws = _Workspace()


def _validate(q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, out, kv_layout, host_io=False):
    """Host-side argument checks the C ABI cannot make from raw pointers: V has
    K's shape/strides/dtype (the library reads V with K's strides), out matches q, the caches
    match q's dtype, metadata is int32 with unit inner stride, and everything lives where the
    call expects it.  Raises PattnError(PATTN_ERR_INVALID_ARG) on any mismatch."""
    if v_cache.shape != k_cache.shape or v_cache.stride() != k_cache.stride():
        raise PattnError(1, "v_cache must have k_cache's shape and strides")
    if k_cache.dtype != q.dtype or v_cache.dtype != q.dtype:
        raise PattnError(1, f"cache dtype {k_cache.dtype}/{v_cache.dtype} != q dtype {q.dtype}")
    if out.shape != q.shape or out.dtype != q.dtype:
        raise PattnError(1, f"out {tuple(out.shape)}/{out.dtype} must match q {tuple(q.shape)}/{q.dtype}")
    if q.dim() != 3 or k_cache.dim() != 4 or block_table.dim() != 2:
        raise PattnError(1, "q must be [T, Hq, D], caches 4-D, block_table 2-D")
    for name, t in (("block_table", block_table), ("cu_seqlens_q", cu_seqlens_q), ("seq_lens", seq_lens)):
        if t.dtype != torch.int32:
            raise PattnError(1, f"{name} must be int32 (got {t.dtype})")
        if t.stride(-1) != 1:
            raise PattnError(1, f"{name} must have unit inner stride")
    B = seq_lens.shape[0]
    if cu_seqlens_q.dim() != 1 or cu_seqlens_q.shape[0] != B + 1 or block_table.shape[0] < B:
        raise PattnError(1, "cu_seqlens_q must have num_seqs + 1 entries and block_table num_seqs rows")
    if not (k_cache.is_cuda and v_cache.is_cuda):
        raise PattnError(1, "k_cache / v_cache must be CUDA tensors")
    dev = k_cache.device
    if v_cache.device != dev:
        raise PattnError(1, "k_cache and v_cache on different devices")
    rest = (q, out, block_table, cu_seqlens_q, seq_lens)
    if host_io:
        if any(t.is_cuda for t in rest):
            raise PattnError(1, "hostio: q, out and the metadata must be host tensors")
        if not all(t.is_contiguous() for t in rest):
            raise PattnError(1, "hostio: q, out and the metadata must be contiguous")
    elif any(t.device != dev for t in rest):
        raise PattnError(1, "all tensors must be on the caches' CUDA device")


def workspace_size(problem: Problem) -> int:
    n = load().pattn_workspace_size(ctypes.byref(problem))
    if n == 0:
        raise PattnError(1, "pattn_workspace_size")
    return int(n)


def unified_attention(
    q: torch.Tensor,
    k_cache: torch.Tensor,
    v_cache: torch.Tensor,
    block_table: torch.Tensor,
    cu_seqlens_q: torch.Tensor,
    seq_lens: torch.Tensor,
    scale: float,
    num_kv_heads: int,
    block_size: int,
    out: Optional[torch.Tensor] = None,
    *,
    kv_layout: str = "NHD",
    max_query_len: Optional[int] = None,
    max_seq_len: Optional[int] = None,
    flags: int = 0,
    workspace: Optional[torch.Tensor] = None,
    stream: Optional[torch.cuda.Stream] = None,
    stream2: Optional[torch.cuda.Stream] = None,
    events: Optional[Sequence[Optional[torch.cuda.Event]]] = None,
) -> torch.Tensor:
    """Unified paged attention over a mixed prefill/decode batch (see include/pattn.h).

    q [T, Hq, D]; k_cache / v_cache [num_blocks, block_size, Hkv, D] ("NHD") or
    [num_blocks, Hkv, block_size, D] ("HND"); block_table int32 [B, max_blocks];
    cu_seqlens_q int32 [B+1]; seq_lens int32 [B] (context + query).  All on one CUDA
    device.  Enqueued on `stream` (default: current); returns `out` without syncing.
    """
    lib = load()
    if out is None:
        out = torch.empty_like(q)
    _validate(q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, out, kv_layout)
    B = seq_lens.shape[0]
    p = make_problem(q, k_cache, num_kv_heads, block_size, block_table, B, out, kv_layout, max_query_len,
                     max_seq_len, flags)
    need = workspace_size(p)
    s = stream if stream is not None else torch.cuda.current_stream(q.device)
    if workspace is None:
        ws = _ws.get(need, q.device, s)  # per (device, stream); never freed while a graph may use it
    else:
        ws = workspace
        if ws.numel() < need:
            raise PattnError(6, f"workspace of {ws.numel()} bytes < {need}")
    args = (
        ctypes.byref(p), q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), block_table.data_ptr(),
        cu_seqlens_q.data_ptr(), seq_lens.data_ptr(), ctypes.c_float(scale), out.data_ptr(), ws.data_ptr(),
        ws.numel(), s.cuda_stream,
    )
    if stream2 is None and events is None:
        _check(lib.pattn_unified_attention(*args), "pattn_unified_attention")
    else:
        o = ExecOpts()
        o.stream2 = stream2.cuda_stream if stream2 is not None else None
        if events is not None:
            for i, e in enumerate(events):
                o.events[i] = e.cuda_event if e is not None else None
        _check(lib.pattn_unified_attention_ex(*args, ctypes.byref(o)), "pattn_unified_attention_ex")
    return out


def unified_attention_hostio(
    q_host: torch.Tensor,
    k_cache: torch.Tensor,
    v_cache: torch.Tensor,
    block_table_host: torch.Tensor,
    cu_seqlens_q_host: torch.Tensor,
    seq_lens_host: torch.Tensor,
    scale: float,
    num_kv_heads: int,
    block_size: int,
    out_host: torch.Tensor,
    *,
    kv_layout: str = "NHD",
    max_query_len: Optional[int] = None,
    max_seq_len: Optional[int] = None,
    flags: int = 0,
    workspace: Optional[torch.Tensor] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """End-to-end call: q / metadata / out are (pinned) HOST tensors, the caches are on the device.
    The H2D copies, the attention and the D2H copy are enqueued on `stream`; sync before reading out_host."""
    lib = load()
    _validate(q_host, k_cache, v_cache, block_table_host, cu_seqlens_q_host, seq_lens_host, out_host, kv_layout,
              host_io=True)
    B = seq_lens_host.shape[0]
    p = make_problem(q_host, k_cache, num_kv_heads, block_size, block_table_host, B, out_host, kv_layout,
                     max_query_len, max_seq_len, flags)
    need = int(lib.pattn_hostio_workspace_size(ctypes.byref(p)))
    if need == 0:
        raise PattnError(1, "pattn_hostio_workspace_size")
    s = stream if stream is not None else torch.cuda.current_stream(k_cache.device)
    ws = workspace if workspace is not None else _ws.get(need, k_cache.device, s)
    _check(
        lib.pattn_unified_attention_hostio(
            ctypes.byref(p), q_host.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), block_table_host.data_ptr(),
            cu_seqlens_q_host.data_ptr(), seq_lens_host.data_ptr(), ctypes.c_float(scale), out_host.data_ptr(),
            ws.data_ptr(), ws.numel(), s.cuda_stream,
        ),
        "pattn_unified_attention_hostio",
    )
    return out_host


class Graph:
    """A captured unified call (pattn_graph_capture): replay with launch(); the tensors given
    at capture are baked in -- refresh their contents between launches."""

    def __init__(self, handle: int, keep: tuple):
        self.handle = handle
        self._keep = keep  # the captured buffers must outlive the graph

    def launch(self, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream()
        _check(load().pattn_graph_launch(self.handle, s.cuda_stream), "pattn_graph_launch")

    def close(self):
        if self.handle:
            _check(load().pattn_graph_destroy(self.handle), "pattn_graph_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def graph_capture(q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, scale, num_kv_heads, block_size, out,
                  workspace, *, kv_layout="NHD", max_query_len=None, max_seq_len=None, flags=0,
                  stream: Optional[torch.cuda.Stream] = None, stream2: Optional[torch.cuda.Stream] = None) -> Graph:
    """Capture one unified call on the given (persistent) buffers into a CUDA graph (PAPER.md
    §6.2).  `workspace` is required: it is baked into the graph."""
    lib = load()
    _validate(q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, out, kv_layout)
    p = make_problem(q, k_cache, num_kv_heads, block_size, block_table, seq_lens.shape[0], out, kv_layout,
                     max_query_len, max_seq_len, flags)
    need = workspace_size(p)
    if workspace.numel() < need:
        raise PattnError(6, f"workspace of {workspace.numel()} bytes < {need}")
    s = stream if stream is not None else torch.cuda.Stream(q.device)
    h = ctypes.c_void_p()
    _check(lib.pattn_graph_capture(
        ctypes.byref(p), q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), block_table.data_ptr(),
        cu_seqlens_q.data_ptr(), seq_lens.data_ptr(), ctypes.c_float(scale), out.data_ptr(), workspace.data_ptr(),
        workspace.numel(), s.cuda_stream, stream2.cuda_stream if stream2 is not None else None, ctypes.byref(h)),
        "pattn_graph_capture")
    return Graph(h.value, (q, k_cache, v_cache, block_table, cu_seqlens_q, seq_lens, out, workspace, s, stream2))


def write_kv(
    k_new: torch.Tensor,
    v_new: torch.Tensor,
    k_cache: torch.Tensor,
    v_cache: torch.Tensor,
    block_table: torch.Tensor,
    cu_seqlens_q: torch.Tensor,
    seq_lens: torch.Tensor,
    block_size: int,
    *,
    kv_layout: str = "NHD",
    stream: Optional[torch.cuda.Stream] = None,
) -> None:
    """Paged KV write (pattn_write_kv): store k_new / v_new [T, Hkv, D] rows of the batch's query
    tokens into the caches at positions ctx_b + i through the block table.  Enqueued on `stream`."""
    lib = load()
    if k_new.shape != v_new.shape or k_new.stride() != v_new.stride() or k_new.stride(2) != 1:
        raise PattnError(1, "k_new/v_new shape/stride mismatch")
    if k_cache.shape != v_cache.shape or k_cache.stride() != v_cache.stride():
        raise PattnError(1, "k_cache/v_cache shape/stride mismatch")
    if k_new.dtype != k_cache.dtype:
        raise PattnError(1, "dtype mismatch")
    T, hkv, _ = k_new.shape
    p = make_problem(k_new, k_cache, hkv, block_size, block_table, seq_lens.shape[0], None, kv_layout)
    s = stream if stream is not None else torch.cuda.current_stream(k_cache.device)
    _check(
        lib.pattn_write_kv(ctypes.byref(p), k_new.data_ptr(), v_new.data_ptr(), k_new.stride(0), k_new.stride(1),
                           k_cache.data_ptr(), v_cache.data_ptr(), block_table.data_ptr(), cu_seqlens_q.data_ptr(),
                           seq_lens.data_ptr(), s.cuda_stream),
        "pattn_write_kv",
    )


def hostio_workspace_size(problem: Problem) -> int:
    """Bytes of device workspace pattn_unified_attention_hostio needs (q/out staging + metadata)."""
    n = load().pattn_hostio_workspace_size(ctypes.byref(problem))
    if n == 0:
        raise PattnError(1, "pattn_hostio_workspace_size")
    return int(n)


def debug_plan(problem: Problem, cu_seqlens_q: torch.Tensor, seq_lens: torch.Tensor) -> torch.Tensor:
    """Run only the metadata kernel K5 and return its plan (int32 device tensor, layout in pattn.h)."""
    lib = load()
    B = problem.num_seqs
    cap = 2 * B + 10
    plan = torch.full((cap,), -7, dtype=torch.int32, device=cu_seqlens_q.device)
    need = workspace_size(problem)
    s = torch.cuda.current_stream(cu_seqlens_q.device)
    ws = _ws.get(need, cu_seqlens_q.device, s)
    _check(
        lib.pattn_debug_plan(ctypes.byref(problem), cu_seqlens_q.data_ptr(), seq_lens.data_ptr(), plan.data_ptr(), cap,
                             ws.data_ptr(), ws.numel(), s.cuda_stream),
        "pattn_debug_plan",
    )
    return plan


def validate_metadata_host(problem: Problem, cu_seqlens_q, seq_lens, block_table) -> int:
    """Host-side metadata validation (SPEC error taxonomy); inputs are CPU int32 tensors/arrays."""
    import numpy as np

    lib = load()
    cu = np.ascontiguousarray(cu_seqlens_q, np.int32)
    sl = np.ascontiguousarray(seq_lens, np.int32)
    bt = np.ascontiguousarray(block_table, np.int32)
    i32p = ctypes.POINTER(ctypes.c_int32)
    return int(lib.pattn_validate_metadata_host(ctypes.byref(problem), cu.ctypes.data_as(i32p),
                                                sl.ctypes.data_as(i32p), bt.ctypes.data_as(i32p)))


def planned_launches(problem: Problem) -> int:
    return int(load().pattn_planned_launches(ctypes.byref(problem)))


def planned_kernels(problem: Problem) -> int:
    """Bit mask of kernel kinds (1 << KERNEL_*) the call launches."""
    return int(load().pattn_planned_kernels(ctypes.byref(problem)))


def make_events(n_steps: int):
    """Per-step lists of 2*KERNEL_COUNT timing events for the `events=` option.  Each event is
    recorded once here so torch materialises it; the library re-records it around its kernel."""
    out = []
    for _ in range(n_steps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * KERNEL_COUNT)]
        for e in evs:
            e.record()
        out.append(evs)
    return out


def workspace_prefill_sms(workspace: torch.Tensor) -> int:
    """K1's SM count chosen by K5 in the last call that used `workspace` (header word
    kHdrPrefillCtas): the two-stream partition, or all SMs when serial.  Reads 4
    bytes device->host (synchronous); for reporting only, never on the hot path."""
    return int(workspace[28:32].view(torch.int32).item())


def version() -> int:
    return int(load().pattn_version())
