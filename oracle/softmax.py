"""The paper's tiled (online) softmax and parallel-tiled-softmax segment merge, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Followed step by step, in the paper's order:

* Tiled softmax, §4.1 "Tiled Softmax": each score row is
  partitioned into tiles processed incrementally; the state is the running
  maximum m, the running sum of exponentials l and the (unnormalised) output
  accumulator acc; when the maximum changes the intermediate results are
  rescaled; the division by l is delayed to the end.
* Parallel tiled softmax, §4.5 (App. C): tiles are grouped
  into segments; each segment runs the iterative tiled softmax on its own and
  stores (acc, m, l); a reduction step combines and rescales the segment
  results "in a manner analogous to the iterative tiled softmax".
* Segment assignment: contiguous tile ranges, ceil(num_tiles / S) tiles per
  segment, trailing segments possibly empty (reading R9; the paper's
  only example is 32 tiles -> 4 segments x 8 tiles).

A segment with no visible key keeps m = -inf, l = 0 and is skipped by the merge
(SPEC S:198).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

State = Tuple[np.ndarray, np.ndarray, np.ndarray]  # (m [r], l [r], acc [r, D])


def init_state(rows: int, head_dim: int) -> State:
    """Before any tile: m = -inf, l = 0, acc = 0."""
    return (np.full(rows, -np.inf), np.zeros(rows), np.zeros((rows, head_dim)))


def online_update(state: State, s_tile: np.ndarray, v_tile: np.ndarray, mask: np.ndarray) -> State:
    """One tile of the tiled softmax.

    s_tile [r, t] scores, v_tile [t, D], mask [r, t] True where the key is visible.
    m' = max(m, max_visible s); alpha = e^{m - m'}; p = e^{s - m'} (0 where masked);
    l' = alpha*l + sum p; acc' = alpha*acc + p @ V.  Rows with no visible key are unchanged.
    """
    m, l, acc = state
    s = np.where(mask, s_tile, -np.inf)
    m_new = np.maximum(m, s.max(axis=1))
    live = np.isfinite(m_new)
    with np.errstate(invalid="ignore"):  # (-inf) - (-inf) only on rows with no visible key yet
        alpha = np.where(live, np.exp(np.where(live, m - m_new, 0.0)), 1.0)
    p = np.where(mask, np.exp(s - np.where(live, m_new, 0.0)[:, None]), 0.0)
    l_new = alpha * l + p.sum(axis=1)
    # masked keys contribute exactly nothing (their V rows are never multiplied)
    v = np.where(mask.any(axis=0)[:, None], v_tile, 0.0)
    acc_new = alpha[:, None] * acc + p @ v
    return (m_new, l_new, acc_new)


def finalize(state: State) -> np.ndarray:
    """out = acc / l (the delayed division).  l == 0 -> EmptyAttentionRow."""
    m, l, acc = state
    if np.any(l <= 0):
        raise ValueError("EmptyAttentionRow")
    return acc / l[:, None]


def tile_ranges(n_keys: int, tile: int) -> List[Tuple[int, int]]:
    return [(s, min(n_keys, s + tile)) for s in range(0, n_keys, tile)]


def assign_tiles_to_segments(num_tiles: int, num_segments: int) -> List[Tuple[int, int]]:
    """Contiguous tile ranges [start, end) per segment; ceil(num_tiles/S) tiles each (reading R9)."""
    if num_segments < 1:
        raise ValueError("InvalidConfig")
    per = -(-num_tiles // num_segments) if num_tiles else 0
    out = []
    for s in range(num_segments):
        a = min(num_tiles, s * per)
        b = min(num_tiles, a + per)
        out.append((a, b))
    return out


def tiled_attention(q_rows, K, V, scale, visible, tiles: Sequence[Tuple[int, int]]):
    """Iterative tiled softmax over the given key tiles (any sizes, in order).

    q_rows [r, D]; K, V [n, D]; visible[i] = number of keys row i sees (prefix, self-inclusive)."""
    r, D = q_rows.shape
    st = init_state(r, D)
    for a, b in tiles:
        s = scale * (q_rows @ K[a:b].T)
        mask = np.arange(a, b)[None, :] < np.asarray(visible)[:, None]
        st = online_update(st, s, V[a:b], mask)
    return st


def segment_partials(q_rows, K, V, scale, visible, tiles, segments) -> List[State]:
    """Each segment runs the tiled softmax over its own tiles and stores (m, l, acc)."""
    return [tiled_attention(q_rows, K, V, scale, visible, tiles[a:b]) for a, b in segments]


def merge_segments(parts: Sequence[State]) -> np.ndarray:
    """Reduction of segment results: M = max_s m_s; w_s = e^{m_s - M} (0 for empty
    segments); out = sum_s w_s acc_s / sum_s w_s l_s."""
    ms = np.stack([p[0] for p in parts])  # [S, r]
    M = ms.max(axis=0)
    if np.any(~np.isfinite(M)):
        raise ValueError("EmptyAttentionRow")
    num = np.zeros_like(parts[0][2])
    den = np.zeros_like(parts[0][1])
    for m, l, acc in parts:
        w = np.where(np.isfinite(m), np.exp(np.where(np.isfinite(m), m - M, 0.0)), 0.0)
        num += w[:, None] * acc
        den += w * l
    return num / den[:, None]
