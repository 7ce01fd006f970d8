#!/usr/bin/env python
"""GPU micro-benchmark sweep -> tuning records -> fitted decision tree (§4.2
P:104-118 two-step flow; SPEC tuner S:375-463; host logic in paper_2511_11581_b200/tuner.py).

  python scripts/tune.py [--out profiles/r01] [--warmup 20 --iters 100] [--depth 3]

For every scenario (synthetic batch of varying batch size, context and prompt lengths,
Llama-class GQA heads) and every planner configuration of the grid, the unified call is
timed with CUDA events (the paper's protocol: 20 warm-up, mean of 100), after
checking that the configuration's output equals the default configuration's within the
bf16 tolerance (tuning never changes the math).  Records go to <out>/tuning_records.ndjson,
the fitted tree to <out>/tuning_tree.json and paper_2511_11581_b200/tuning_tree.json
(installed by pattn.load()).
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


def scenarios():
    s = []
    for B, ctx in [(1, 8192), (1, 131072), (4, 32768), (8, 131072), (16, 16384), (32, 4096), (64, 4096),
                   (128, 2048), (256, 1024), (256, 4096)]:
        s.append(Workload(f"dec_b{B}_ctx{ctx}", tuple((ctx, 1) for _ in range(B)), 32, 8, 128, 16, "bf16"))
    s.append(Workload("dec70_b8_ctx131072", tuple((131072, 1) for _ in range(8)), 64, 8, 128, 16, "bf16"))
    s.append(CONFIGS["c3_mixed8b"])
    s.append(Workload("mix_2p2048_56d4096", tuple([(0, 2048)] * 2 + [(4096, 1)] * 56), 32, 8, 128, 16, "bf16"))
    s.append(Workload("mix70_4p2048_28d4096", tuple([(0, 2048)] * 4 + [(4096, 1)] * 28), 64, 8, 128, 16, "bf16"))
    s.append(Workload("mix_8p512_120d8192", tuple([(0, 512)] * 8 + [(8192, 1)] * 120), 32, 8, 128, 16, "bf16"))
    return s


GRID = [dict(zip(tuner.KNOBS, v)) for v in itertools.product([4, 8, 16, 32], [128, 256, 1024, 4096], [1, 2, 3, 4])]


def features(w):
    return {"num_seqs": w.num_seqs, "num_tokens": w.num_tokens, "max_query_len": max(q for _, q in w.seqs),
            "max_seq_len": max(c + q for c, q in w.seqs)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01"))
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--depth", type=int, default=4)
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    rec_path = os.path.join(args.out, "tuning_records.ndjson")
    if os.path.exists(rec_path):
        os.remove(rec_path)
    pattn.load()
    tuner.install(None)
    dev = torch.device("cuda", 0)
    s1 = torch.cuda.current_stream(dev)
    s2 = torch.cuda.Stream(dev)
    for w in scenarios():
        inp = generate_device(w, seed=7, device=dev)
        q, kc, vc = inp["q"], inp["k_cache"], inp["v_cache"]
        bt, cu, sl = inp["block_table"], inp["cu_seqlens_q"], inp["seq_lens"]
        f = features(w)
        out = torch.empty_like(q)

        def call():
            pattn.unified_attention(q, kc, vc, bt, cu, sl, w.scale, w.num_kv_heads, w.block_size, out,
                                    max_query_len=f["max_query_len"], max_seq_len=f["max_seq_len"], stream=s1,
                                    stream2=s2)

        tuner.install(None)
        call()
        torch.cuda.synchronize()
        ref = out.float().clone()
        recs = []
        for cfg in GRID:
            tuner.install(cfg)
            out.zero_()
            call()
            torch.cuda.synchronize()
            err = (out.float() - ref).abs()
            ok = bool(torch.isfinite(out.float()).all()) and bool((err <= 1e-2 + 1e-2 * ref.abs()).all())
            for _ in range(args.warmup):
                call()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.iters)]
            for e0, e1 in evs:
                e0.record(s1)
                call()
                e1.record(s1)
            torch.cuda.synchronize()
            lat = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
            rec = {"scenario": w.name, "features": f, "config": cfg, "iterations": args.iters,
                   "latency_us": {"mean": statistics.fmean(lat), "p50": lat[len(lat) // 2],
                                  "p95": lat[min(len(lat) - 1, int(0.95 * len(lat)))]},
                   "matches_default": ok}
            if not ok:
                rec["latency_us"]["mean"] = float("inf")  # never selectable
            recs.append(rec)
        tuner.write_records(rec_path, recs)
        best = min(recs, key=lambda r: r["latency_us"]["mean"])
        dflt = [r for r in recs if r["config"] == {"items_per_sm": 16, "min_chunk_tokens": 256,
                                                     "decode_ctas_per_sm": 2}]
        print(f"{w.name:28s} best {best['latency_us']['mean']:9.1f} us {best['config']}"
              + (f"  (default-like 16/256/2: {dflt[0]['latency_us']['mean']:.1f})" if dflt else ""), flush=True)
        del inp, q, kc, vc, out, ref
        torch.cuda.empty_cache()
    tuner.install(None)
    recs = tuner.read_records(rec_path)
    tree = tuner.fit_decision_tree(recs, max_depth=args.depth)
    print(tuner.to_pseudocode(tree))
    print("training regret: tree %.1f us, best single config %.1f us" %
          (tuner.tree_regret(tree, recs), tuner.best_global_regret(recs)))
    for path in (os.path.join(args.out, "tuning_tree.json"), os.path.join(ROOT, "paper_2511_11581_b200",
                                                                          "tuning_tree.json")):
        json.dump(tree, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
