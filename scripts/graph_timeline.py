"""Eager call vs CUDA-graph replay of the same mixed step: per-kernel CTA timelines (trace build).

  PATTN_LIB=variants/trace/libpattn.so python scripts/graph_timeline.py [workload]

For K1 and the decode kernel K2W: CTAs recorded (CTAs that leave at once through the SM partition
record nothing), SMs used, first / last CTA start and end relative to the step's first CTA, and
how many CTAs started late (after K1's first wave).  Debug tooling only (globaltimer)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_11581_b200 import pattn  # noqa: E402
from workloads import CONFIGS  # noqa: E402
from workloads.gen import generate_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3_mixed8b"
w = CONFIGS[name]
inp = generate_device(w, seed=1, device="cuda")
out = torch.empty_like(inp["q"])
lib = pattn.load()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
mq, ml = max(q for _, q in w.seqs), max(c + q for c, q in w.seqs)
p = pattn.make_problem(inp["q"], inp["k_cache"], w.num_kv_heads, w.block_size, inp["block_table"], w.num_seqs, out,
                       "NHD", mq, ml)
ws = torch.empty(pattn.workspace_size(p), dtype=torch.uint8, device="cuda")


def eager():
    with torch.cuda.stream(s1):
        pattn.unified_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_table"], inp["cu_seqlens_q"],
                                inp["seq_lens"], w.scale, w.num_kv_heads, w.block_size, out, max_query_len=mq,
                                max_seq_len=ml, workspace=ws, stream=s1, stream2=s2)


def spans():
    res = {}
    for k in ("k1", "k2w"):
        fn = getattr(lib, f"pattn_debug_{k}_cta", None)
        if fn is None:
            continue
        buf = (ctypes.c_ulonglong * (4 * 2048))()
        fn(buf, 2048)
        res[k] = np.array(buf[:], dtype=np.uint64).reshape(2048, 4).astype(np.int64)
    return res


def report(tag, before):
    after = spans()
    t0 = None
    rows = {}
    for k, a in after.items():
        fresh = (a[:, 0] != before[k][:, 0]) & (a[:, 0] > 0)  # CTAs written by this launch
        rows[k] = a[fresh]
        if fresh.any():
            m = int(a[fresh, 0].min())
            t0 = m if t0 is None else min(t0, m)
    for k, a in rows.items():
        if len(a) == 0:
            print(f"{tag} {k}: no CTAs recorded")
            continue
        st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
        print(f"{tag} {k}: {len(a)} CTAs on {len(np.unique(a[:, 2]))} SMs; start {st.min():7.1f} .. {st.max():7.1f} us;"
              f" end {en.min():7.1f} .. {en.max():7.1f} us; CTAs starting > 20 us late: {(st > 20).sum()}")


for _ in range(3):
    eager()
torch.cuda.synchronize()
b = spans()
eager()
torch.cuda.synchronize()
report("eager", b)

g = pattn.graph_capture(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_table"], inp["cu_seqlens_q"],
                        inp["seq_lens"], w.scale, w.num_kv_heads, w.block_size, out, ws, max_query_len=mq,
                        max_seq_len=ml, stream=s1, stream2=s2)
for _ in range(3):
    g.launch(s1)
torch.cuda.synchronize()
for rep in range(3):
    b = spans()
    g.launch(s1)
    torch.cuda.synchronize()
    report(f"graph{rep}", b)
