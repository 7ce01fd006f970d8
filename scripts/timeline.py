"""SM timeline of one unified call (trace build):
  PATTN_LIB=variants/trace/libpattn.so python scripts/timeline.py [workload] [streams] [seqs_override]
Prints per-kernel CTA spans (globaltimer), SMs busy per kernel over time, and for the decode
kernel's CTA 0 the per-sub-block producer->consumer latencies (clock64)."""
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
streams = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = CONFIGS[name]
if len(sys.argv) > 3:
    seqs = []
    for grp in sys.argv[3].split("+"):
        n, rest = grp.split("x")
        ctx, q = rest.split(":")
        seqs += [(int(ctx), int(q))] * int(n)
    w = w.with_seqs(seqs, name=name + "_x")
inp = generate_device(w, seed=1, device="cuda")
out = torch.empty_like(inp["q"])
lib = pattn.load()
s2 = torch.cuda.Stream() if streams == 2 else None


def call():
    pattn.unified_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_table"], inp["cu_seqlens_q"],
                            inp["seq_lens"], w.scale, w.num_kv_heads, w.block_size, out,
                            max_query_len=max(q for _, q in w.seqs), max_seq_len=max(c + q for c, q in w.seqs),
                            stream2=s2)


ev_buf = (ctypes.c_ulonglong * (8 * 4096))()
for _ in range(3):
    call()
torch.cuda.synchronize()
if hasattr(lib, "pattn_debug_k2_ev"):
    lib.pattn_debug_k2_ev(ev_buf, 8 * 4096, 1)
call()
torch.cuda.synchronize()

spans = {}
for k in ("k1", "k2"):
    fn = getattr(lib, f"pattn_debug_{k}_cta", None)
    if fn is None:
        continue
    buf = (ctypes.c_ulonglong * (4 * 2048))()
    fn(buf, 2048)
    a = np.array(buf[:], dtype=np.uint64).reshape(2048, 4).astype(np.int64)
    spans[k] = a
t0 = min(int(a[a[:, 0] > 0, 0].min()) for a in spans.values() if (a[:, 0] > 0).any())
# keep only CTAs of the last launch (those starting within 5 ms of the earliest)
for k, a in spans.items():
    live = (a[:, 0] >= t0) & (a[:, 0] < t0 + 5_000_000)
    a = a[live]
    spans[k] = a
    if len(a) == 0:
        print(k, "no CTAs")
        continue
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    print(f"{k}: {len(a)} CTAs on {len(np.unique(a[:, 2]))} SMs, start {st.min():.1f}-{st.max():.1f} us, "
          f"end {en.min():.1f}-{en.max():.1f} us, items/CTA min {a[:, 3].min()} max {a[:, 3].max()} "
          f"mean {a[:, 3].mean():.1f}")
    late = st > 5
    if late.any():
        print(f"   {late.sum()} CTAs started late (>5us): starts {np.percentile(st[late], [0, 50, 100]).round(1)}")
T = max(((a[:, 1] - t0).max() / 1e3) for a in spans.values() if len(a))
print(f"span {T:.1f} us; SMs busy per 25 us bin (k1 / k2):")
for b0 in np.arange(0, T, 25.0):
    row = []
    for k, a in spans.items():
        st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
        on = (st < b0 + 25) & (en > b0)
        row.append(len(np.unique(a[on, 2])))
    print(f"  {b0:6.0f} us  " + " / ".join(str(r) for r in row))

if hasattr(lib, "pattn_debug_k2_ev"):
    lib.pattn_debug_k2_ev(ev_buf, 8 * 4096, 1)
    ev = np.array(ev_buf[:], dtype=np.uint64).reshape(8, 4096).astype(np.int64)
    issue, wait, ready, done = ev[0], ev[1], ev[2], ev[3]
    ok = (issue > 0) & (wait > 0) & (ready > 0) & (done > 0)
    gs = np.nonzero(ok)[0]
    if len(gs):
        lat, stall, comp = ready[gs] - issue[gs], ready[gs] - wait[gs], done[gs] - ready[gs]
        iss = np.diff(issue[gs])
        print(f"k2 CTA0: {len(gs)} sub-blocks; clk: issue->ready p50 {np.median(lat):.0f} p90 "
              f"{np.percentile(lat, 90):.0f}; consumer wait p50 {np.median(stall):.0f} mean {stall.mean():.0f}; "
              f"compute p50 {np.median(comp):.0f} mean {comp.mean():.0f}; issue spacing p50 {np.median(iss):.0f} "
              f"mean {iss.mean():.0f}")
        it0, it1 = ev[4], ev[5]
        k = np.nonzero((it0 > 0) & (it1 > 0))[0]
        if len(k) > 1:
            print(f"   items {len(k)}: item span p50 {np.median(it1[k] - it0[k]):.0f} clk, gap end->next start p50 "
                  f"{np.median(it0[k[1:]] - it1[k[:-1]]):.0f} clk")
