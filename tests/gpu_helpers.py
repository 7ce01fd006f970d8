"""Shared helpers for the GPU parity tests: upload a workloads.Batch, call libpattn through
its C ABI (paper_2511_11581_b200.pattn), compare with the oracle element by element."""
from __future__ import annotations

import numpy as np
import torch

from paper_2511_11581_b200 import pattn

BF16_ATOL = 1e-2  # north_star: max |err| <= 1e-2 abs + 1e-2 rel (bf16 inputs, fp32 accumulation)
BF16_RTOL = 1e-2
F32_ATOL = 1e-5  # north_star: <= 1e-5 for the fp32 path
F32_RTOL = 1e-5


def to_torch(a: np.ndarray, device="cuda") -> torch.Tensor:
    if a.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(device).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


class DeviceBatch:
    def __init__(self, batch, device="cuda"):
        self.batch = batch
        self.q = to_torch(batch.q, device)
        self.k = to_torch(batch.k_cache, device)
        self.v = to_torch(batch.v_cache, device)
        self.bt = torch.from_numpy(batch.block_table).to(device)
        self.cu = torch.from_numpy(batch.cu_seqlens_q).to(device)
        self.sl = torch.from_numpy(batch.seq_lens).to(device)

    def run(self, flags=0, out=None, **kw):
        w = self.batch.workload
        qlens = np.diff(self.batch.cu_seqlens_q)
        o = pattn.unified_attention(
            self.q, self.k, self.v, self.bt, self.cu, self.sl, w.scale, w.num_kv_heads, w.block_size, out,
            kv_layout=self.batch.layout, max_query_len=int(qlens.max()) if len(qlens) else 0,
            max_seq_len=int(self.batch.seq_lens.max()), flags=flags, **kw,
        )
        torch.cuda.synchronize()
        return o


def out_f64(o: torch.Tensor) -> np.ndarray:
    return o.float().cpu().numpy().astype(np.float64)


def assert_close(gpu: np.ndarray, ref: np.ndarray, dtype: str, what: str = ""):
    atol, rtol = (F32_ATOL, F32_RTOL) if dtype == "f32" else (BF16_ATOL, BF16_RTOL)
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    assert np.isfinite(gpu).all(), f"{what}: non-finite output"
    err = np.abs(gpu - ref)
    bound = atol + rtol * np.abs(ref)
    bad = err > bound
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(
            f"{what}: {bad.sum()} / {bad.size} elements out of tolerance; max abs err {err.max():.3e}; "
            f"first {idx.tolist()} gpu={gpu[tuple(idx[0])]} ref={ref[tuple(idx[0])]}"
        )
    return float(err.max())
