"""Seeded paged-attention batch generator (input recipe: DESIGN.md §3).

Recipe (SURVEY.md §8(d) "Synthetic inputs", extending SPEC S:465-504):
  * numpy PCG64(seed); Q, K, V ~ U[-1, 1] in fp32, rounded
    round-to-nearest-even to the workload dtype.  Both the oracle and the GPU
    see exactly the rounded values.
  * physical block ids are a seeded permutation of [0, num_blocks); sequences
    take their blocks in order; num_blocks = sum(ceil(L_b/bs)) + spare.
  * block_table rows are padded with -1; unused blocks and the slots t >= L_b of
    each sequence's last block hold NaN ("poison", reading R13) so a
    kernel that reads outside the visible range produces NaN.
  * distributions: "uniform" (above), "peaked" (q scaled x8 before rounding: a
    sharper softmax), "needle" (K = 0 except one row per (seq, kv head) = +4,
    q = +4: one key dominates by >100 nats so the output is that key's V row
    exactly), "zero_q" (q = 0: all scores equal).

No attention arithmetic lives here.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

BF16_NAN = np.uint16(0x7FC0)


# ----------------------------------------------------------------------------
# dtype conversion (storage only)
# ----------------------------------------------------------------------------
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern, round-to-nearest-even (NaN stays NaN)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    nan = np.isnan(x)
    rounding = ((u >> 16) & 1) + np.uint32(0x7FFF)
    out = ((u + rounding) >> 16).astype(np.uint16)
    if nan.any():
        out[nan] = BF16_NAN
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """bf16 bit pattern -> fp32 (exact)."""
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ----------------------------------------------------------------------------
# workloads (BASELINE.json configs; readings in DESIGN.md §3 / SURVEY §8(c) #18)
# ----------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    seqs: Tuple[Tuple[int, int], ...]  # (context_len, query_len) per sequence
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    block_size: int
    dtype: str  # "f32" | "bf16" | "f16"

    @property
    def scale(self) -> float:
        # 1/sqrt(d_k) (Eq. 1) rounded to the fp32 scalar the ABI takes.
        return float(np.float32(1.0 / math.sqrt(self.head_dim)))

    @property
    def num_tokens(self) -> int:
        return sum(q for _, q in self.seqs)

    @property
    def num_seqs(self) -> int:
        return len(self.seqs)

    def with_seqs(self, seqs, name=None) -> "Workload":
        return dataclasses.replace(self, seqs=tuple(tuple(s) for s in seqs), name=name or self.name)

    def algorithmic(self) -> Dict[str, float]:
        """Algorithmic work: causally visible (row,key) pairs only."""
        D, Hq, Hkv, bs = self.head_dim, self.num_q_heads, self.num_kv_heads, self.block_size
        esz = 4 if self.dtype == "f32" else 2
        flops_prefill = flops_decode = 0.0
        kv_prefill = kv_decode = 0.0
        for ctx, q in self.seqs:
            L = ctx + q
            visible = q * ctx + q * (q + 1) / 2  # sum_i (ctx + i + 1)
            f = 4.0 * D * Hq * visible
            kvb = L * Hkv * 2 * D * esz + math.ceil(L / bs) * 4
            if q == 1:
                flops_decode += f
                kv_decode += kvb
            else:
                flops_prefill += f
                kv_prefill += kvb
        qo = 2.0 * self.num_tokens * Hq * D * esz
        return dict(
            flops=flops_prefill + flops_decode,
            flops_prefill=flops_prefill,
            flops_decode=flops_decode,
            bytes=kv_prefill + kv_decode + qo,
            bytes_kv_decode=kv_decode,
            bytes_kv_prefill=kv_prefill,
            bytes_qo=qo,
            bytes_decode=kv_decode + 2.0 * sum(1 for _, q in self.seqs if q == 1) * Hq * D * esz,
        )


CONFIGS: Dict[str, Workload] = {
    # 1. tiny paged attention: 1 prefill of 16 tokens + 1 decode with 32-token context; 4 Q / 1 KV, d 64, bs 16, fp32
    "c1_tiny": Workload("c1_tiny", ((0, 16), (32, 1)), 4, 1, 64, 16, "f32"),
    # 2. Llama-3.1-8B decode: 64 x (ctx 4096, q 1), 32/8 heads, d 128, bs 16, bf16
    "c2_decode8b": Workload("c2_decode8b", tuple((4096, 1) for _ in range(64)), 32, 8, 128, 16, "bf16"),
    # 3. Llama-3.1-8B mixed: 8 prefills of 2k + 56 decodes at 4k context, one unified call
    "c3_mixed8b": Workload(
        "c3_mixed8b", tuple([(0, 2048)] * 8 + [(4096, 1)] * 56), 32, 8, 128, 16, "bf16"
    ),
    # 4. long-context decode: 8 x (ctx 131072, q 1), GQA 8:1 (64 Q / 8 KV), d 128
    "c4_decode128k": Workload("c4_decode128k", tuple((131072, 1) for _ in range(8)), 64, 8, 128, 16, "bf16"),
    # 5. Llama-3.1-70B mixed, 256 seqs = 32 x (ctx 0, q 2048) + 224 x (ctx 4096, q 1)
    "c5_mixed70b": Workload(
        "c5_mixed70b", tuple([(0, 2048)] * 32 + [(4096, 1)] * 224), 64, 8, 128, 16, "bf16"
    ),
}
# Phase-attribution workloads (not BASELINE configs): each half of config 3 on its own.
ATTRIBUTION: Dict[str, Workload] = {
    "c3p_prefill_part": CONFIGS["c3_mixed8b"].with_seqs([(0, 2048)] * 8, name="c3p_prefill_part"),
    "c3d_decode_part": CONFIGS["c3_mixed8b"].with_seqs([(4096, 1)] * 56, name="c3d_decode_part"),
    # shapes outside the BASELINE configs that exercise the widened kernel envelope (bench lines)
    # GQA 7:1 (28 query / 4 KV heads, e.g. Qwen2-7B): the tcgen05 prefill with padding rows
    "x_g7_mixed": Workload("x_g7_mixed", tuple([(0, 2048)] * 8 + [(4096, 1)] * 56), 28, 4, 128, 16, "bf16"),
    # head_dim 64 (32 / 8 heads): the D = 64 instantiation of the tcgen05 prefill kernel
    "x_d64_mixed": Workload("x_d64_mixed", tuple([(0, 2048)] * 8 + [(4096, 1)] * 56), 32, 8, 64, 16, "bf16"),
    # block size 7 (not a multiple of 16): long decodes split on K2W with cp.async-gathered rows, merged by K3
    "x_bs7_decode32k": Workload("x_bs7_decode32k", tuple((32768, 1) for _ in range(8)), 32, 8, 128, 7, "bf16"),
    # GQA 12:1 decode (96 query / 8 KV heads, e.g. Mistral-Large): K2W with two head groups per KV head
    "x_g12_decode8k": Workload("x_g12_decode8k", tuple((8192, 1) for _ in range(32)), 96, 8, 128, 16, "bf16"),
    # config 3's mix with block size 7: K1 and K2W gather K/V rows with cp.async (no TMA box fits a page)
    "x_bs7_mixed": Workload("x_bs7_mixed", tuple([(0, 2048)] * 8 + [(4096, 1)] * 56), 32, 8, 128, 7, "bf16"),
}


# ----------------------------------------------------------------------------
# batch
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Batch:
    workload: Workload
    layout: str  # "NHD": [num_blocks, bs, Hkv, D]; "HND": [num_blocks, Hkv, bs, D]
    q: np.ndarray  # [T, Hq, D]  float32 (f32), uint16 bf16 bits (bf16) or float16 (f16)
    k_cache: np.ndarray
    v_cache: np.ndarray
    block_table: np.ndarray  # int32 [B, max_blocks_per_seq], padded with -1
    cu_seqlens_q: np.ndarray  # int32 [B+1]
    seq_lens: np.ndarray  # int32 [B]  (= context + query)
    needle_pos: Optional[np.ndarray] = None  # int64 [B, Hkv] for dist="needle"

    @property
    def num_blocks(self) -> int:
        return int(self.k_cache.shape[0])

    @property
    def dtype(self) -> str:
        return self.workload.dtype

    def kv_strides(self) -> Tuple[int, int, int]:
        """(stride_blk, stride_tok, stride_head) in elements."""
        w = self.workload
        if self.layout == "NHD":
            return (w.block_size * w.num_kv_heads * w.head_dim, w.num_kv_heads * w.head_dim, w.head_dim)
        return (w.num_kv_heads * w.block_size * w.head_dim, w.head_dim, w.block_size * w.head_dim)

    def as_f32(self, a: np.ndarray) -> np.ndarray:
        return bf16_bits_to_f32(a) if a.dtype == np.uint16 else a


def _uniform(rng: np.random.Generator, shape, dtype: str, mult: float = 1.0) -> np.ndarray:
    """U[-1,1]*mult drawn in fp32, rounded to the storage dtype (chunked to bound memory)."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.uint16 if dtype == "bf16" else (np.float16 if dtype == "f16" else np.float32))
    chunk = 1 << 24
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        x = rng.random(e - s, dtype=np.float32)
        x *= np.float32(2.0 * mult)
        x -= np.float32(mult)
        # fp16: numpy's float32 -> float16 cast rounds to nearest even
        out[s:e] = f32_to_bf16_bits(x) if dtype == "bf16" else x.astype(out.dtype)
    return out.reshape(shape)


def _const(shape, value: float, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return np.full(shape, f32_to_bf16_bits(np.array([value], np.float32))[0], dtype=np.uint16)
    if dtype == "f16":
        return np.full(shape, value, dtype=np.float16)
    return np.full(shape, value, dtype=np.float32)


def generate(
    w: Workload,
    seed: int,
    dist: str = "uniform",
    poison: bool = True,
    layout: str = "NHD",
    spare_blocks: int = 8,
    permute_blocks: bool = True,
    needle_pos: Optional[Sequence[Sequence[int]]] = None,
) -> Batch:
    rng = np.random.Generator(np.random.PCG64(seed))
    B, Hq, Hkv, D, bs = w.num_seqs, w.num_q_heads, w.num_kv_heads, w.head_dim, w.block_size
    assert Hq % Hkv == 0
    q_lens = np.array([q for _, q in w.seqs], dtype=np.int64)
    seq_lens = np.array([c + q for c, q in w.seqs], dtype=np.int64)
    nblk = (seq_lens + bs - 1) // bs
    num_blocks = int(nblk.sum()) + spare_blocks
    max_blocks = max(1, int(nblk.max()) if B else 1)
    T = int(q_lens.sum())

    cu = np.zeros(B + 1, dtype=np.int32)
    cu[1:] = np.cumsum(q_lens)

    perm = rng.permutation(num_blocks).astype(np.int32) if permute_blocks else np.arange(num_blocks, dtype=np.int32)
    bt = np.full((B, max_blocks), -1, dtype=np.int32)
    off = 0
    for b in range(B):
        bt[b, : nblk[b]] = perm[off : off + nblk[b]]
        off += int(nblk[b])

    dt = w.dtype
    # logical NHD cache
    kv_shape = (num_blocks, bs, Hkv, D)
    qmult = 8.0 if dist == "peaked" else 1.0
    if dist == "zero_q":
        q = _const((T, Hq, D), 0.0, dt)
    elif dist == "needle":
        q = _const((T, Hq, D), 4.0, dt)
    else:
        q = _uniform(rng, (T, Hq, D), dt, qmult)
    if dist == "needle":
        k = _const(kv_shape, 0.0, dt)
    else:
        k = _uniform(rng, kv_shape, dt)
    v = _uniform(rng, kv_shape, dt)

    npos = None
    if dist == "needle":
        if needle_pos is None:
            npos = np.zeros((B, Hkv), dtype=np.int64)
            for b in range(B):
                ctx = w.seqs[b][0]
                # visible to every query row of the sequence: position < ctx + 1
                npos[b] = rng.integers(0, max(1, ctx + 1), size=Hkv)
        else:
            npos = np.asarray(needle_pos, dtype=np.int64).reshape(B, Hkv)
        four = _const((D,), 4.0, dt)
        for b in range(B):
            for g in range(Hkv):
                t = int(npos[b, g])
                k[bt[b, t // bs], t % bs, g, :] = four

    if poison:
        nan = BF16_NAN if dt == "bf16" else (np.float16(np.nan) if dt == "f16" else np.float32(np.nan))
        used = np.zeros(num_blocks, dtype=bool)
        for b in range(B):
            used[bt[b, : nblk[b]]] = True
            tail = int(seq_lens[b] % bs)
            if tail:
                last = bt[b, nblk[b] - 1]
                k[last, tail:] = nan
                v[last, tail:] = nan
        k[~used] = nan
        v[~used] = nan

    if layout == "HND":
        k = np.ascontiguousarray(k.transpose(0, 2, 1, 3))
        v = np.ascontiguousarray(v.transpose(0, 2, 1, 3))
    elif layout != "NHD":
        raise ValueError(layout)

    return Batch(
        workload=w,
        layout=layout,
        q=q,
        k_cache=k,
        v_cache=v,
        block_table=bt,
        cu_seqlens_q=cu,
        seq_lens=seq_lens.astype(np.int32),
        needle_pos=npos,
    )


def generate_device(w: Workload, seed: int, device="cuda", layout: str = "NHD", spare_blocks: int = 8):
    """Same structure as generate() (U[-1,1] values rounded to the dtype, permuted physical
    blocks, -1 padded block table) drawn with torch's generator directly on the device, for
    the large bench workloads.  Unused cache slots hold finite values (timing runs).
    Returns a dict of device tensors plus host copies of the metadata."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    B, Hq, Hkv, D, bs = w.num_seqs, w.num_q_heads, w.num_kv_heads, w.head_dim, w.block_size
    q_lens = torch.tensor([q for _, q in w.seqs], dtype=torch.int64)
    seq_lens = torch.tensor([c + q for c, q in w.seqs], dtype=torch.int64)
    nblk = (seq_lens + bs - 1) // bs
    num_blocks = int(nblk.sum()) + spare_blocks
    max_blocks = max(1, int(nblk.max()))
    T = int(q_lens.sum())
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16}.get(w.dtype, torch.float32)

    def uni(shape):
        out = torch.empty(shape, dtype=tdt, device=device)
        flat = out.view(-1)
        chunk = 1 << 27
        for s in range(0, flat.numel(), chunk):
            e = min(flat.numel(), s + chunk)
            x = torch.rand(e - s, generator=g, device=device, dtype=torch.float32)
            flat[s:e] = (x * 2.0 - 1.0).to(tdt)
        return out

    kv_shape = (num_blocks, bs, Hkv, D) if layout == "NHD" else (num_blocks, Hkv, bs, D)
    q = uni((T, Hq, D))
    k = uni(kv_shape)
    v = uni(kv_shape)
    perm = torch.randperm(num_blocks, generator=g, device=device).to(torch.int32).cpu()
    bt = torch.full((B, max_blocks), -1, dtype=torch.int32)
    off = 0
    for b in range(B):
        n = int(nblk[b])
        bt[b, :n] = perm[off : off + n]
        off += n
    cu = torch.zeros(B + 1, dtype=torch.int32)
    cu[1:] = torch.cumsum(q_lens, 0).to(torch.int32)
    return dict(
        q=q, k_cache=k, v_cache=v,
        block_table=bt.to(device), cu_seqlens_q=cu.to(device), seq_lens=seq_lens.to(torch.int32).to(device),
        block_table_h=bt, cu_seqlens_q_h=cu, seq_lens_h=seq_lens.to(torch.int32),
        layout=layout, num_blocks=num_blocks,
    )


def random_workload(
    rng: np.random.Generator,
    heads: Tuple[int, int],
    head_dim: int,
    block_size: int,
    dtype: str,
    max_seqs: int = 6,
    max_len: int = 300,
    decode_share: float = 0.5,
    name: str = "random",
) -> Workload:
    """Ragged mixed batch: decodes (q=1, ctx>=0), prefills (ctx=0) and chunked prefills (ctx>0, q>1)."""
    B = int(rng.integers(1, max_seqs + 1))
    seqs: List[Tuple[int, int]] = []
    for _ in range(B):
        if rng.random() < decode_share:
            seqs.append((int(rng.integers(0, max_len)), 1))
        elif rng.random() < 0.5:
            seqs.append((0, int(rng.integers(2, max_len + 1))))
        else:
            seqs.append((int(rng.integers(1, max_len)), int(rng.integers(2, max_len // 2 + 2))))
    return Workload(name, tuple(seqs), heads[0], heads[1], head_dim, block_size, dtype)
