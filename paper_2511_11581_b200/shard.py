"""Multi-GPU batch sharder for unified paged attention.

Attention has no exchange between (sequence, KV head) units (Q blocks never span
sequences or KV heads; segments merge only within a unit), so a
batch shards with NO collective on the data path:

  * mode "seq":    rank r gets a subset of whole sequences (data-parallel attention);
                   balanced by greedy LPT on a per-sequence cost
                   c_b = prefill_flops_b / F + kv_bytes_b / BW (class-aware: compute-bound
                   prefills and HBM-bound decodes weigh on different roofs).
  * mode "kvhead": rank r owns KV heads [r*Hkv/P, (r+1)*Hkv/P) and their G*Hkv/P query
                   heads for every sequence (the tensor-parallel shape).

Each rank then calls libpattn on its local batch.  `gather_outputs` (NCCL or gloo
all-gather) is used only for verification, outside timed regions.

Host logic is plain numpy/torch; it never imports oracle/.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np
import torch

# B200 roofs used only to weigh prefill vs decode work in the balancer (measured peaks)
F_PEAK = 1.6e15  # bf16 flop/s
BW_PEAK = 6.5e12  # HBM byte/s


@dataclasses.dataclass
class ShardPlan:
    mode: str
    world: int
    seq_ids: List[np.ndarray]  # per rank: global sequence ids (mode "seq"); all ids (mode "kvhead")
    kv_heads: List[range]  # per rank: owned KV heads
    q_heads: List[range]  # per rank: owned query heads
    cost: np.ndarray  # per rank: balanced cost (seconds at peak)


def sequence_costs(q_lens: np.ndarray, seq_lens: np.ndarray, num_q_heads: int, num_kv_heads: int, head_dim: int,
                   esz: int = 2) -> np.ndarray:
    q = q_lens.astype(np.float64)
    L = seq_lens.astype(np.float64)
    ctx = L - q
    visible = q * ctx + q * (q + 1) / 2.0
    flops = 4.0 * head_dim * num_q_heads * visible
    kv_bytes = L * num_kv_heads * 2.0 * head_dim * esz
    return flops / F_PEAK + kv_bytes / BW_PEAK


def plan_shards(cu_seqlens_q: np.ndarray, seq_lens: np.ndarray, num_q_heads: int, num_kv_heads: int, head_dim: int,
                world: int, mode: str = "seq") -> ShardPlan:
    cu = np.asarray(cu_seqlens_q, np.int64)
    sl = np.asarray(seq_lens, np.int64)
    B = len(sl)
    q_lens = np.diff(cu)
    G = num_q_heads // num_kv_heads
    if mode == "kvhead":
        if num_kv_heads % world:
            raise ValueError("kvhead sharding needs num_kv_heads % world == 0")
        per = num_kv_heads // world
        kvh = [range(r * per, (r + 1) * per) for r in range(world)]
        qh = [range(r * per * G, (r + 1) * per * G) for r in range(world)]
        c = sequence_costs(q_lens, sl, num_q_heads, num_kv_heads, head_dim).sum() / world
        return ShardPlan(mode, world, [np.arange(B)] * world, kvh, qh, np.full(world, c))
    if mode != "seq":
        raise ValueError(mode)
    cost = sequence_costs(q_lens, sl, num_q_heads, num_kv_heads, head_dim)
    order = np.argsort(-cost, kind="stable")  # longest processing time first
    load = np.zeros(world)
    owner = np.empty(B, np.int64)
    for b in order:
        r = int(np.argmin(load))  # ties -> lowest rank (deterministic)
        owner[b] = r
        load[r] += cost[b]
    ids = [np.sort(np.nonzero(owner == r)[0]) for r in range(world)]
    return ShardPlan(mode, world, ids, [range(num_kv_heads)] * world, [range(num_q_heads)] * world, load)


@dataclasses.dataclass
class LocalBatch:
    q: torch.Tensor
    k_cache: torch.Tensor
    v_cache: torch.Tensor
    block_table: torch.Tensor
    cu_seqlens_q: torch.Tensor
    seq_lens: torch.Tensor
    token_ids: np.ndarray  # global token index of each local token
    num_kv_heads: int
    q_heads: range


def local_batch(plan: ShardPlan, rank: int, q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                block_table: np.ndarray, cu_seqlens_q: np.ndarray, seq_lens: np.ndarray, block_size: int,
                device: Optional[torch.device] = None, kv_layout: str = "NHD") -> LocalBatch:
    """Build rank `rank`'s local inputs from global ones.  Caches are NHD
    [num_blocks, block_size, Hkv, D] or HND [num_blocks, Hkv, block_size, D] (`kv_layout`).
    Mode "seq": the rank's sequences, their blocks gathered into a compact local cache and the
    block table renumbered 0..n-1.  Mode "kvhead": the rank's KV-head slice of the caches and
    query-head slice of q."""
    if kv_layout not in ("NHD", "HND"):
        raise ValueError(kv_layout)
    head_axis = 2 if kv_layout == "NHD" else 1
    dev = device if device is not None else q.device
    cu = np.asarray(cu_seqlens_q, np.int64)
    sl = np.asarray(seq_lens, np.int64)
    bt = np.asarray(block_table)
    if plan.mode == "kvhead":
        kvh, qh = plan.kv_heads[rank], plan.q_heads[rank]
        return LocalBatch(
            q=q[:, qh.start:qh.stop].contiguous().to(dev),
            k_cache=k_cache.narrow(head_axis, kvh.start, len(kvh)).contiguous().to(dev),
            v_cache=v_cache.narrow(head_axis, kvh.start, len(kvh)).contiguous().to(dev),
            block_table=torch.from_numpy(bt.astype(np.int32)).to(dev),
            cu_seqlens_q=torch.from_numpy(cu.astype(np.int32)).to(dev),
            seq_lens=torch.from_numpy(sl.astype(np.int32)).to(dev),
            token_ids=np.arange(cu[-1]),
            num_kv_heads=len(kvh),
            q_heads=qh,
        )
    ids = plan.seq_ids[rank]
    nblk = (sl[ids] + block_size - 1) // block_size
    blocks = np.concatenate([bt[b, :n] for b, n in zip(ids, nblk)]) if len(ids) else np.zeros(0, np.int64)
    maxb = int(nblk.max()) if len(ids) else 1
    lbt = np.full((max(1, len(ids)), max(1, maxb)), -1, np.int32)
    off = 0
    for i, n in enumerate(nblk):
        lbt[i, :n] = np.arange(off, off + n)
        off += int(n)
    tok = np.concatenate([np.arange(cu[b], cu[b + 1]) for b in ids]) if len(ids) else np.zeros(0, np.int64)
    lcu = np.zeros(len(ids) + 1, np.int32)
    lcu[1:] = np.cumsum(cu[ids + 1] - cu[ids]) if len(ids) else []
    bidx = torch.from_numpy(blocks.astype(np.int64)).to(k_cache.device)
    tidx = torch.from_numpy(tok.astype(np.int64)).to(q.device)
    return LocalBatch(
        q=q.index_select(0, tidx).to(dev),
        k_cache=k_cache.index_select(0, bidx).to(dev),
        v_cache=v_cache.index_select(0, bidx).to(dev),
        block_table=torch.from_numpy(lbt).to(dev),
        cu_seqlens_q=torch.from_numpy(lcu).to(dev),
        seq_lens=torch.from_numpy(sl[ids].astype(np.int32)).to(dev),
        token_ids=tok,
        num_kv_heads=k_cache.shape[head_axis],
        q_heads=range(q.shape[1]),
    )


def rank_token_ids(plan: ShardPlan, r: int, cu_seqlens_q: Sequence[int]) -> np.ndarray:
    """Global token ids of rank r's local tokens (every rank can compute every rank's ids)."""
    cu = np.asarray(cu_seqlens_q, np.int64)
    ids = plan.seq_ids[r]
    if not len(ids):
        return np.zeros(0, np.int64)
    return np.concatenate([np.arange(cu[b], cu[b + 1]) for b in ids])


def gather_outputs(plan: ShardPlan, local_out: torch.Tensor, cu_seqlens_q: Sequence[int], num_q_heads: int,
                   group=None) -> torch.Tensor:
    """All-gather every rank's local output and scatter it into global [T, Hq, D] order.
    Verification only (untimed).  Works with NCCL (CUDA tensors) and gloo (CPU tensors)."""
    import torch.distributed as dist

    world = plan.world
    D = local_out.shape[-1]
    num_tokens = int(np.asarray(cu_seqlens_q)[-1])
    if plan.mode == "kvhead":
        parts = [torch.empty_like(local_out) for _ in range(world)]
        dist.all_gather(parts, local_out.contiguous(), group=group)
        return torch.cat(parts, dim=1)
    counts = [len(rank_token_ids(plan, r, cu_seqlens_q)) for r in range(world)]
    mx = max(max(counts), 1)
    pad = torch.zeros((mx, num_q_heads, D), dtype=local_out.dtype, device=local_out.device)
    pad[: local_out.shape[0]] = local_out
    gathered = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(gathered, pad, group=group)
    out = torch.empty((num_tokens, num_q_heads, D), dtype=local_out.dtype, device=local_out.device)
    for r in range(world):
        ids = torch.from_numpy(rank_token_ids(plan, r, cu_seqlens_q)).to(out.device)
        out.index_copy_(0, ids, gathered[r][: counts[r]])
    return out
