"""Tuning flow: micro-benchmark records -> fitted if-else decision tree -> libpattn planner.

PAPER.md §4.2: kernels are tuned "outside of the vLLM runtime" with
micro-benchmarks over scenarios of varying context lengths, prompt lengths and batch sizes;
the results are exported "as heuristics --- simple if-else decision trees", which also give
configurations for scenarios that were not benchmarked.  SPEC's tuner module
fixes the artefacts: an NDJSON records file (schema "v": 1) and a JSON tree with internal
nodes {"feature", "threshold", "lt", "ge"} and leaves holding a configuration.

Here a configuration is the planner's launch knobs (pattn_tuning_t, include/pattn.h):
  items_per_sm        decode work items (segment x KV head x head group) per SM  -> segment count
  min_chunk_tokens    shortest decode segment, in keys
  decode_ctas_per_sm  resident decode CTAs per SM
  k2_sm_mbs           mixed batches: the per-SM decode rate K5's SM-partition model assumes
                      (shifts SMs between the concurrent prefill and decode kernels)
  serial              mixed batches: prefill and decode back to back instead of concurrent
  decode_kernel       1 = K2W (head-wide TMA boxes, where it applies), 2 = K2 (one KV head per item)
(0 = the built-in default for any knob).
and the features are the host-known batch quantities the planner sees (PATTN_FEAT_*):
num_seqs, num_tokens, max_query_len (1 = decode-only batch), max_seq_len.

The fitter is greedy and top-down: at each node it picks the (feature, threshold) split that
minimises the summed latency regret of giving every scenario in a child that child's best
single configuration; it stops at max_depth or when no split lowers the regret.  Host logic
only (numpy); the GPU sweep that produces the records is scripts/tune.py.
"""
from __future__ import annotations

import ctypes
import json
import math
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

FEATURES = ["num_seqs", "num_tokens", "max_query_len", "max_seq_len"]  # order = PATTN_FEAT_*
KNOBS = ["items_per_sm", "min_chunk_tokens", "decode_ctas_per_sm", "k2_sm_mbs", "serial", "decode_kernel"]


# libpattn's built-in value of each knob (used where a tree leaf or record holds 0)
# 0 where the default depends on the decode kernel the planner picks: items_per_sm (K2 16, K2W 2),
# min_chunk_tokens (K2 256, K2W 128),
# k2_sm_mbs (the kernel's measured per-SM rate: K2W 100 GB/s, K2 61 GB/s)
DEFAULTS = {"items_per_sm": 0, "min_chunk_tokens": 0, "decode_ctas_per_sm": 2, "k2_sm_mbs": 0, "serial": 0,
            "decode_kernel": 1}


def with_defaults(cfg: Dict) -> Dict:
    """A configuration with 0 ("built-in default") replaced by the default's value."""
    return {k: int(cfg.get(k, 0)) or DEFAULTS[k] for k in KNOBS}


class NoData(ValueError):
    pass


def config_key(cfg: Dict) -> Tuple[int, ...]:
    return tuple(int(cfg.get(k, 0)) for k in KNOBS)


def _scenario_table(records: Iterable[Dict]):
    """scenario label -> (features, {config key: mean latency})."""
    table: Dict[str, Tuple[Dict, Dict]] = {}
    for r in records:
        lab = r["scenario"]
        feats, lat = table.setdefault(lab, (dict(r["features"]), {}))
        key = config_key(r["config"])
        m = float(r["latency_us"]["mean"])
        lat[key] = min(m, lat.get(key, math.inf))
    return table


def _regret(labels, table, key) -> float:
    """Summed latency regret (us) of running config `key` on every scenario in `labels`
    (a config a scenario did not measure counts as +inf)."""
    tot = 0.0
    for lab in labels:
        lat = table[lab][1]
        tot += lat.get(key, math.inf) - min(lat.values())
    return tot


def _best_config(labels, table):
    keys = sorted({k for lab in labels for k in table[lab][1]})
    best = min(keys, key=lambda k: (_regret(labels, table, k), k))
    return best, _regret(labels, table, best)


def fit_decision_tree(records: Sequence[Dict], max_depth: int = 3, min_gain: float = 0.0) -> Dict:
    """Greedy regret-minimising tree (JSON form).  Raises NoData on empty input.

    min_gain: a split must lower the node's summed regret by at least this fraction of the
    summed best latency of the node's scenarios (a noise floor: run-to-run spread is ~1 %, and a
    split that only chases it does not carry over to unseen scenarios)."""
    table = _scenario_table(records)
    if not table:
        raise NoData("no tuning records")

    def build(labels, depth):
        key, reg = _best_config(labels, table)
        leaf = {k: v for k, v in zip(KNOBS, key)}
        if depth >= max_depth or reg <= 0.0 or len(labels) < 2:
            return leaf
        floor = min_gain * sum(min(table[lab][1].values()) for lab in labels)
        best = None
        for fi, f in enumerate(FEATURES):
            vals = sorted({table[lab][0][f] for lab in labels})
            for lo, hi in zip(vals[:-1], vals[1:]):
                thr = (lo + hi) / 2.0
                lt = [lab for lab in labels if table[lab][0][f] < thr]
                ge = [lab for lab in labels if table[lab][0][f] >= thr]
                r = _best_config(lt, table)[1] + _best_config(ge, table)[1]
                cand = (r, fi, thr)
                if best is None or cand < best:
                    best = (r, fi, thr, lt, ge)
        if best is None or best[0] >= reg or reg - best[0] < floor:
            return leaf
        _, fi, thr, lt, ge = best
        return {"feature": FEATURES[fi], "threshold": thr, "lt": build(lt, depth + 1), "ge": build(ge, depth + 1)}

    return build(sorted(table), 0)


def select(tree: Dict, features: Dict) -> Dict:
    """Leaf configuration for a feature vector (O(depth))."""
    node = tree
    while "feature" in node:
        node = node["lt"] if features[node["feature"]] < node["threshold"] else node["ge"]
    return {k: int(node.get(k, 0)) for k in KNOBS}


def tree_regret(tree: Dict, records: Sequence[Dict]) -> float:
    table = _scenario_table(records)
    return sum(_regret([lab], table, config_key(select(tree, table[lab][0]))) for lab in table)


def best_global_regret(records: Sequence[Dict]) -> float:
    table = _scenario_table(records)
    return _best_config(sorted(table), table)[1]


def depth(tree: Dict) -> int:
    return 0 if "feature" not in tree else 1 + max(depth(tree["lt"]), depth(tree["ge"]))


# ------------------------------------------------------------------ persistence
def write_records(path: str, records: Iterable[Dict]) -> None:
    with open(path, "a") as f:
        for r in records:
            f.write(json.dumps(dict(r, v=1)) + "\n")


def read_records(path: str) -> List[Dict]:
    with open(path) as f:
        return [json.loads(line) for line in f if line.strip()]


def to_pseudocode(tree: Dict, indent: str = "") -> str:
    if "feature" not in tree:
        return indent + "return " + ", ".join(f"{k}={tree.get(k, 0)}" for k in KNOBS) + "\n"
    return (f"{indent}if {tree['feature']} < {tree['threshold']:g}:\n" + to_pseudocode(tree["lt"], indent + "    ")
            + f"{indent}else:\n" + to_pseudocode(tree["ge"], indent + "    "))


# ------------------------------------------------------------------ libpattn (pattn_set_tuning_tree)
class Tuning(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in KNOBS]


class TreeNode(ctypes.Structure):
    _fields_ = [("feature", ctypes.c_int32), ("lt", ctypes.c_int32), ("ge", ctypes.c_int32),
                ("threshold", ctypes.c_double), ("leaf", Tuning)]


def flatten(tree: Dict) -> List[TreeNode]:
    """Pre-order array with the root at 0 and every child after its parent (the ABI's rule)."""
    out: List[Optional[TreeNode]] = []

    def emit(node) -> int:
        i = len(out)
        out.append(None)
        n = TreeNode()
        if "feature" in node:
            n.feature = FEATURES.index(node["feature"])
            n.threshold = float(node["threshold"])
            n.lt = emit(node["lt"])
            n.ge = emit(node["ge"])
        else:
            n.feature = -1
            n.lt = n.ge = 0
            for k in KNOBS:
                setattr(n.leaf, k, int(node.get(k, 0)))
        out[i] = n
        return i

    emit(tree)
    return out  # type: ignore[return-value]


def install(tree: Optional[Dict]) -> None:
    """Load `tree` into libpattn's planner (None removes it)."""
    from . import pattn

    lib = pattn.load()
    if tree is None:
        pattn._check(lib.pattn_set_tuning_tree(None, 0), "pattn_set_tuning_tree")
        return
    nodes = flatten(tree)
    arr = (TreeNode * len(nodes))(*nodes)
    pattn._check(lib.pattn_set_tuning_tree(arr, len(nodes)), "pattn_set_tuning_tree")


def default_tree() -> Optional[Dict]:
    """The committed fitted tree (paper_2511_11581_b200/tuning_tree.json), or None."""
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tuning_tree.json")
    return json.load(open(path)) if os.path.exists(path) else None


def planned_tuning(problem) -> Dict:
    """The knobs libpattn's planner resolves for a problem (host-only, pattn_plan_tuning)."""
    from . import pattn

    lib = pattn.load()
    t = Tuning()
    pattn._check(lib.pattn_plan_tuning(ctypes.byref(problem), ctypes.byref(t)), "pattn_plan_tuning")
    return {k: int(getattr(t, k)) for k in KNOBS}
