#!/usr/bin/env python
"""GPU micro-benchmark sweep -> tuning records -> fitted decision tree -> held-out check
(§4.2 P:104-118 two-step flow; SPEC tuner S:375-463; host logic in
paper_2511_11581_b200/tuner.py).

  python scripts/tune.py [--out profiles/r02] [--warmup 20 --iters 100] [--depth 4]

Scenarios: synthetic batches of varying batch size, context and prompt lengths, Llama-class
GQA heads.  TRAIN scenarios produce the records the tree is fitted on; HOLDOUT scenarios
(other lengths and mixes, never seen by the fitter) measure how the tree generalises -- the
paper's claim that the exported trees give configurations "for scenarios that were not part
of the tuning".

Per scenario the unified call is timed with CUDA events (the paper's protocol: 20
warm-up, mean of 100), after checking that the configuration's output equals the default
configuration's within the bf16 tolerance (tuning never changes the math):
  stage 1  the decode kernel and its knobs (K2W: items_per_sm x min_chunk_tokens, 16 configs;
           K2: items_per_sm x min_chunk_tokens x decode_ctas_per_sm, 64) with the partition
           knobs at their defaults;
  stage 2  mixed batches only: the partition knobs (k2_sm_mbs -- the decode rate per SM that
           K5's SM-partition model assumes -- and serial) at the stage-1 best decode knobs.
           For decode-only batches the partition knobs have no effect; their stage-1 records
           are replicated under every stage-2 value so that the fitter sees them as don't-care.
Records: <out>/tuning_records.ndjson (train), <out>/tuning_records_holdout.ndjson; the fitted
tree: <out>/tuning_tree.json and paper_2511_11581_b200/tuning_tree.json (installed by
pattn.load()); the held-out report: <out>/tuning_holdout.json.
"""
import argparse
import itertools
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_11581_b200 import pattn, tuner  # noqa: E402
from workloads import CONFIGS, Workload  # noqa: E402
from workloads.gen import generate_device  # noqa: E402


def _dec(name, B, ctx, hq=32, hkv=8):
    return Workload(name, tuple((ctx, 1) for _ in range(B)), hq, hkv, 128, 16, "bf16")


def _mix(name, npre, qlen, ndec, ctx, hq=32, hkv=8):
    return Workload(name, tuple([(0, qlen)] * npre + [(ctx, 1)] * ndec), hq, hkv, 128, 16, "bf16")


def train_scenarios():
    s = [_dec(f"dec_b{B}_ctx{ctx}", B, ctx) for B, ctx in
         [(1, 8192), (1, 131072), (4, 32768), (8, 131072), (16, 16384), (32, 4096), (64, 4096), (128, 2048),
          (256, 1024), (256, 4096)]]
    s.append(_dec("dec70_b8_ctx131072", 8, 131072, 64, 8))
    s.append(CONFIGS["c3_mixed8b"])
    s.append(_mix("mix_2p2048_56d4096", 2, 2048, 56, 4096))
    s.append(_mix("mix70_4p2048_28d4096", 4, 2048, 28, 4096, 64, 8))
    s.append(_mix("mix_8p512_120d8192", 8, 512, 120, 8192))
    return s


def holdout_scenarios():
    return [
        _dec("ho_dec_b24_ctx6000", 24, 6000),
        _dec("ho_dec_b2_ctx65536", 2, 65536),
        _dec("ho_dec_b96_ctx3000", 96, 3000),
        _dec("ho_dec70_b16_ctx32768", 16, 32768, 64, 8),
        _mix("ho_mix_4p1024_60d2048", 4, 1024, 60, 2048),
        _mix("ho_mix_1p4096_31d16384", 1, 4096, 31, 16384),
        _mix("ho_mix70_2p3000_40d8192", 2, 3000, 40, 8192, 64, 8),
        _mix("ho_mix_16p256_48d4096", 16, 256, 48, 4096),
    ]


# decode kernel x its knobs: K2W (decode_kernel 1, one CTA per SM) and K2 (2, 1-4 CTAs per SM)
DECODE_GRID = ([{"items_per_sm": i, "min_chunk_tokens": m, "decode_ctas_per_sm": 1, "decode_kernel": 1}
                for i, m in itertools.product([2, 4, 8, 16], [128, 256, 1024, 4096])] +
               [{"items_per_sm": i, "min_chunk_tokens": m, "decode_ctas_per_sm": c, "decode_kernel": 2}
                for i, m, c in itertools.product([4, 8, 16, 32], [128, 256, 1024, 4096], [1, 2, 3, 4])])
PARTITION_GRID = ([{"k2_sm_mbs": v, "serial": 0} for v in (45000, 61000, 80000, 100000, 120000)] +
                  [{"k2_sm_mbs": 0, "serial": 1}])


def full(cfg):
    return {k: int(cfg.get(k, 0)) for k in tuner.KNOBS}


def features(w):
    return {"num_seqs": w.num_seqs, "num_tokens": w.num_tokens, "max_query_len": max(q for _, q in w.seqs),
            "max_seq_len": max(c + q for c, q in w.seqs)}


class Bench:
    def __init__(self, w, dev, s1, s2, warmup, iters):
        self.w, self.s1, self.s2, self.warmup, self.iters = w, s1, s2, warmup, iters
        inp = generate_device(w, seed=7, device=dev)
        self.inp = inp
        self.f = features(w)
        self.out = torch.empty_like(inp["q"])
        tuner.install(None)
        self.call()
        torch.cuda.synchronize()
        self.ref = self.out.float().clone()

    def call(self):
        x, w, f = self.inp, self.w, self.f
        pattn.unified_attention(x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["cu_seqlens_q"],
                                x["seq_lens"], w.scale, w.num_kv_heads, w.block_size, self.out,
                                max_query_len=f["max_query_len"], max_seq_len=f["max_seq_len"], stream=self.s1,
                                stream2=self.s2)

    def record(self, cfg):
        tuner.install(full(cfg))  # a depth-0 tree = this configuration for every batch
        self.out.zero_()
        self.call()
        torch.cuda.synchronize()
        err = (self.out.float() - self.ref).abs()
        ok = bool(torch.isfinite(self.out.float()).all()) and bool((err <= 1e-2 + 1e-2 * self.ref.abs()).all())
        for _ in range(self.warmup):
            self.call()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(self.iters)]
        for e0, e1 in evs:
            e0.record(self.s1)
            self.call()
            e1.record(self.s1)
        torch.cuda.synchronize()
        lat = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
        rec = {"scenario": self.w.name, "features": self.f, "config": full(cfg), "iterations": self.iters,
               "latency_us": {"mean": statistics.fmean(lat), "p50": lat[len(lat) // 2],
                              "p95": lat[min(len(lat) - 1, int(0.95 * len(lat)))]},
               "matches_default": ok}
        if not ok:
            rec["latency_us"]["mean"] = float("inf")  # never selectable
        return rec


def sweep(w, dev, s1, s2, args):
    """Stage 1 + stage 2 records of one scenario."""
    b = Bench(w, dev, s1, s2, args.warmup, args.iters)
    recs = [b.record(c) for c in DECODE_GRID]
    best = min(recs, key=lambda r: r["latency_us"]["mean"])["config"]
    if b.f["max_query_len"] > 1:
        recs += [b.record(dict(best, **pc)) for pc in PARTITION_GRID]
    else:  # partition knobs are don't-care without a prefill kernel
        extra = []
        for r in recs:
            for pc in PARTITION_GRID:
                extra.append(dict(r, config=dict(r["config"], **pc), replicated=True))
        recs += extra
    return b, recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02"))
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--depth", type=int, default=4)
    ap.add_argument("--min-gain", type=float, default=0.005,
                    help="a split must cut the node's regret by this fraction of its summed best latency")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    paths = {k: os.path.join(args.out, f"tuning_records{k}.ndjson") for k in ("", "_holdout")}
    for p in paths.values():
        if os.path.exists(p):
            os.remove(p)
    pattn.load()
    dev = torch.device("cuda", 0)
    s1 = torch.cuda.current_stream(dev)
    s2 = torch.cuda.Stream(dev)
    for w in train_scenarios():
        b, recs = sweep(w, dev, s1, s2, args)
        tuner.write_records(paths[""], recs)
        best = min(recs, key=lambda r: r["latency_us"]["mean"])
        print(f"train   {w.name:28s} best {best['latency_us']['mean']:9.1f} us {best['config']}", flush=True)
        del b
        torch.cuda.empty_cache()
    train = tuner.read_records(paths[""])
    tree = tuner.fit_decision_tree(train, max_depth=args.depth, min_gain=args.min_gain)
    unreg = tuner.fit_decision_tree(train, max_depth=args.depth)  # for the report: the unregularised fit
    print(tuner.to_pseudocode(tree))
    report = {"train": {"scenarios": len({r["scenario"] for r in train}),
                        "tree_depth": tuner.depth(tree), "min_gain": args.min_gain,
                        "unregularised_tree_depth": tuner.depth(unreg),
                        "unregularised_tree_regret_us": tuner.tree_regret(unreg, train),
                        "tree_regret_us": tuner.tree_regret(tree, train),
                        "best_single_config_regret_us": tuner.best_global_regret(train)},
              "holdout": []}
    # held-out scenarios: their own full sweep (to know the best), plus the tree's choice
    best_single = tuner.fit_decision_tree(train, max_depth=0)
    for w in holdout_scenarios():
        b, recs = sweep(w, dev, s1, s2, args)
        choice = full(tuner.select(tree, features(w)))
        single = full(best_single)
        unreg_choice = full(tuner.select(unreg, features(w)))
        for c in (choice, single, unreg_choice, full({})):
            if all(r["config"] != c for r in recs):  # (replicated decode-only records count: exact)
                recs.append(b.record(c))
        tuner.write_records(paths["_holdout"], recs)
        table = {tuner.config_key(r["config"]): r["latency_us"]["mean"] for r in recs}
        best = min(table.values())
        dflt = table.get(tuner.config_key(full({})), float("nan"))
        entry = {"scenario": w.name, "features": features(w), "best_us": best,
                 "tree_choice": choice, "tree_us": table[tuner.config_key(choice)],
                 "unregularised_tree_us": table[tuner.config_key(unreg_choice)],
                 "best_single_train_config_us": table[tuner.config_key(single)], "default_us": dflt}
        entry["tree_regret_us"] = entry["tree_us"] - best
        report["holdout"].append(entry)
        print(f"holdout {w.name:28s} best {best:9.1f} us  tree {entry['tree_us']:9.1f}  "
              f"best-single {entry['best_single_train_config_us']:9.1f}  default {dflt:9.1f}", flush=True)
        del b
        torch.cuda.empty_cache()
    ho = report["holdout"]
    report["holdout_summary"] = {
        "scenarios": len(ho), "tree_regret_us": sum(e["tree_regret_us"] for e in ho),
        "unregularised_tree_regret_us": sum(e["unregularised_tree_us"] - e["best_us"] for e in ho),
        "best_single_train_config_regret_us": sum(e["best_single_train_config_us"] - e["best_us"] for e in ho),
        "default_regret_us": sum(e["default_us"] - e["best_us"] for e in ho),
        "sum_best_us": sum(e["best_us"] for e in ho)}
    print(json.dumps(report["holdout_summary"]))
    json.dump(report, open(os.path.join(args.out, "tuning_holdout.json"), "w"), indent=1)
    open(os.path.join(args.out, "tuning_tree.txt"), "w").write(tuner.to_pseudocode(tree))
    for path in (os.path.join(args.out, "tuning_tree.json"), os.path.join(ROOT, "paper_2511_11581_b200",
                                                                          "tuning_tree.json")):
        json.dump(tree, open(path, "w"), indent=1)
    tuner.install(tree)


if __name__ == "__main__":
    main()
