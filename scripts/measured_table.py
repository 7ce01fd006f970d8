"""Markdown table of the bench lines in profiles/<round>/bench_*.json (for DESIGN.md §7 and
BASELINE.md).   python scripts/measured_table.py r02"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
print("| workload | step (eager) | CUDA-graph replay | value (tokens/s) | e2e (tokens/s) | dominant roof | other roof |")
print("|---|---|---|---|---|---|---|")
for path in sorted(glob.glob(os.path.join(ROOT, "profiles", rnd, "bench_*.json"))):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    if "impl" in d:
        continue
    name = os.path.basename(path)[6:-5]
    g = (d.get("cuda_graph") or {}).get("ms_per_step")
    e = (d.get("e2e") or {}).get("value")
    rl = d.get("roofline_kernels", {})
    dom = d.get("roofline") or {}

    def fmt(r):
        if not r or r.get("frac") is None:
            return "—"
        extra = f" (share of its {r['prefill_sms']} SMs: {r['frac_of_sm_share']:.2f})" if "frac_of_sm_share" in r else ""
        return f"{r['kernel']} {r['achieved']:.0f} {r['unit']} = {r['frac']:.3f} ({r['bound']}){extra}"

    key = next((k for k, r in rl.items() if r.get("bound") == dom.get("bound") and r.get("achieved") == dom.get("achieved")),
               None)
    domr = rl.get(key, dom)
    others = [fmt(r) for k, r in rl.items() if k != key]
    print(f"| {name} | {d['ms_per_step']:.4f} ms | {g and f'{g:.4f} ms' or '—'} | {d['value']:.3g} | "
          f"{e and f'{e:.3g}' or '—'} | {fmt(domr)} | {'; '.join(others) or '—'} |")
