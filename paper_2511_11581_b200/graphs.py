"""Batch-size-bucketed CUDA graphs of the unified call (§6.2, §4.7).

The paper's "full graph" execution records one graph per batch-size bucket at startup and
replays the bucket that fits each batch; its kernels' frozen launch grids then carry "excess
instances" for smaller batches.  libpattn's grids are persistent and sized from the SM count,
never from the batch, so one recording serves every batch up to the bucket's capacity: the
metadata is device-resident and sequences with q_b = 0 pad the bucket (they produce no rows
and no work items -- only K5 reads them).

This module holds host orchestration only: it owns the static buffers the graphs were
captured on, copies each batch's q / metadata into them (with padding) and launches the
graph through the C ABI (pattn_graph_capture / pattn_graph_launch).  No attention arithmetic.
"""
from __future__ import annotations

from typing import Dict, Optional, Sequence

import torch

from . import pattn


class GraphBuckets:
    """Graphs of pattn_unified_attention for batch sizes up to each bucket (default: powers of
    two up to 128), all over the same paged KV caches.

    max_query_len: largest q_b a batch may carry (1 = decode-only buckets); a bucket of B
    sequences has room for B * max_query_len query tokens unless token_capacity is given.
    max_seq_len: largest L_b (sizes the block-table width and the planner hint)."""

    def __init__(self, k_cache: torch.Tensor, v_cache: torch.Tensor, num_q_heads: int, num_kv_heads: int,
                 block_size: int, scale: float, *, buckets: Sequence[int] = (1, 2, 4, 8, 16, 32, 64, 128),
                 max_query_len: int = 1, max_seq_len: int, token_capacity: Optional[Dict[int, int]] = None,
                 kv_layout: str = "NHD", two_streams: bool = True, flags: int = 0):
        self.k, self.v = k_cache, v_cache
        self.dev = k_cache.device
        self.Hq, self.Hkv, self.bs, self.scale = num_q_heads, num_kv_heads, block_size, scale
        self.D = k_cache.shape[-1]
        self.layout, self.flags = kv_layout, flags
        self.max_q, self.max_L = max_query_len, max_seq_len
        self.max_blocks = (max_seq_len + block_size - 1) // block_size
        self.buckets = sorted(buckets)
        self.stream = torch.cuda.Stream(self.dev)
        self.stream2 = torch.cuda.Stream(self.dev) if two_streams else None
        self.bufs: Dict[int, dict] = {}
        self.graphs: Dict[int, pattn.Graph] = {}
        for B in self.buckets:
            T = (token_capacity or {}).get(B, B * max_query_len)
            b = dict(
                q=torch.zeros((T, num_q_heads, self.D), dtype=k_cache.dtype, device=self.dev),
                out=torch.zeros((T, num_q_heads, self.D), dtype=k_cache.dtype, device=self.dev),
                bt=torch.zeros((B, self.max_blocks), dtype=torch.int32, device=self.dev),
                cu=torch.zeros(B + 1, dtype=torch.int32, device=self.dev),
                sl=torch.zeros(B, dtype=torch.int32, device=self.dev),
            )
            p = pattn.make_problem(b["q"], k_cache, num_kv_heads, block_size, b["bt"], B, b["out"], kv_layout,
                                   max_query_len, max_seq_len, flags)
            b["ws"] = torch.empty(pattn.workspace_size(p), dtype=torch.uint8, device=self.dev)
            self.bufs[B] = b
            self.graphs[B] = pattn.graph_capture(
                b["q"], k_cache, v_cache, b["bt"], b["cu"], b["sl"], scale, num_kv_heads, block_size, b["out"],
                b["ws"], kv_layout=kv_layout, max_query_len=max_query_len, max_seq_len=max_seq_len, flags=flags,
                stream=self.stream, stream2=self.stream2)
        torch.cuda.synchronize(self.dev)

    def bucket_for(self, num_seqs: int, num_tokens: int) -> int:
        for B in self.buckets:
            if B >= num_seqs and self.bufs[B]["q"].shape[0] >= num_tokens:
                return B
        raise ValueError(f"no bucket holds {num_seqs} sequences / {num_tokens} tokens")

    def run(self, q: torch.Tensor, block_table: torch.Tensor, cu_seqlens_q: torch.Tensor, seq_lens: torch.Tensor,
            *, bucket: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """One batch through its bucket's graph: copy q and the metadata into the bucket's
        buffers (padding sequences get q_b = 0, L_b = 0), replay, return out[:T] (a view of the
        bucket's output buffer, valid until the bucket is replayed again)."""
        B, T = seq_lens.shape[0], q.shape[0]
        cap = bucket if bucket is not None else self.bucket_for(B, T)
        b = self.bufs[cap]
        if cap < B or b["q"].shape[0] < T or block_table.shape[1] > self.max_blocks:
            raise ValueError("batch does not fit the bucket")
        s = stream if stream is not None else torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(s):
            b["q"][:T].copy_(q, non_blocking=True)
            b["bt"][:B, : block_table.shape[1]].copy_(block_table, non_blocking=True)
            b["cu"][: B + 1].copy_(cu_seqlens_q, non_blocking=True)
            b["cu"][B + 1:].fill_(T)  # padding sequences: q_b = 0 ...
            b["sl"][:B].copy_(seq_lens, non_blocking=True)
            b["sl"][B:].zero_()  # ... and L_b = 0 (no keys, no blocks read)
        self.graphs[cap].launch(s)
        return b["out"][:T]

    def close(self):
        for g in self.graphs.values():
            g.close()
        self.graphs.clear()
