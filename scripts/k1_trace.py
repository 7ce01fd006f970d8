"""Timeline of K1 on CTA 0 (trace build: make EXTRA=-DPATTN_TRACE), config 3.
  PATTN_LIB=variants/trace/libpattn.so python scripts/k1_trace.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_11581_b200 import pattn  # noqa: E402
from workloads import CONFIGS  # noqa: E402
from workloads.gen import generate_device  # noqa: E402

w = CONFIGS["c3_mixed8b"]
inp = generate_device(w, seed=1, device="cuda")
out = torch.empty_like(inp["q"])
lib = pattn.load()
lib.pattn_debug_k1_trace.restype = ctypes.c_int
buf = (ctypes.c_ulonglong * (2 * 8192))()


def call():
    pattn.unified_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_table"], inp["cu_seqlens_q"],
                            inp["seq_lens"], w.scale, w.num_kv_heads, w.block_size, out, max_query_len=2048,
                            max_seq_len=4097)


for _ in range(3):
    call()
torch.cuda.synchronize()
lib.pattn_debug_k1_trace(buf, 8192, 1)
call()
torch.cuda.synchronize()
n = lib.pattn_debug_k1_trace(buf, 8192, 1)
ev = np.array(buf[: 2 * n], dtype=np.uint64).reshape(n, 2)
ev = ev[np.argsort(ev[:, 0], kind="stable")]
ev = ev[ev[:, 0] > 0]
t0 = ev[0, 0]
names = {1: "K_ready", 2: "V_ready", 3: "Pa_ready", 4: "Pb_ready", 5: "PVa_issued", 6: "PVb_issued", 7: "Sa_issued",
         8: "Sb_issued", 10: "SMa_start", 11: "SMb_start", 12: "SMa_done", 13: "SMb_done", 20: "K_load", 21: "V_load", 22: "K_issued", 23: "V_issued", 30: "SMa_ldS", 31: "SMb_ldS", 32: "SMa_max", 33: "SMb_max", 34: "SMa_exp", 35: "SMb_exp", 40: "item_start", 41: "Q_ready", 42: "EPa_start", 43: "EPb_start", 44: "EPa_done", 45: "EPb_done", 24: "K_wait", 25: "V_wait"}
print("events", n)
for t, c in ev[:160]:
    print(f"{int(t - t0):8d}  {names.get(int(c), c)}")
# a window around the 6th item start (steady state)
starts = np.nonzero(ev[:, 1] == 40)[0]
if len(starts) > 6:
    i0 = starts[5]
    print("---- window around item 6")
    for t, c in ev[max(0, i0 - 60): i0 + 60]:
        print(f"{int(t - t0):8d}  {names.get(int(c), c)}")
# per-event-type mean intervals
for c in sorted(set(ev[:, 1].tolist())):
    ts = ev[ev[:, 1] == c, 0].astype(np.int64)
    if len(ts) > 2:
        d = np.diff(ts)
        print(f"{str(names.get(c, c)):12s} n={len(ts):5d} mean interval {d.mean():8.0f}  median {np.median(d):8.0f}")
sa = ev[ev[:, 1] == 10, 0].astype(np.int64)
da = ev[ev[:, 1] == 12, 0].astype(np.int64)
m = min(len(sa), len(da))
print("softmax a duration median", np.median(da[:m] - sa[:m]))
# where does the MMA thread wait?  gap from the previous MMA event to each readiness event
mma_codes = {1, 2, 3, 4, 5, 6, 7, 8}
mm = ev[np.isin(ev[:, 1], list(mma_codes))]
gaps = {}
for i in range(1, len(mm)):
    c = int(mm[i, 1])
    gaps.setdefault(c, []).append(int(mm[i, 0]) - int(mm[i - 1, 0]))
for c, g in sorted(gaps.items()):
    print(f"MMA gap before {str(names.get(c, c)):12s} median {np.median(g):7.0f} mean {np.mean(g):7.0f}")

for a, b, nm in ((20, 22, "K"), (21, 23, "V")):
    ta = ev[ev[:, 1] == a, 0].astype(np.int64)
    tb = ev[ev[:, 1] == b, 0].astype(np.int64)
    m = min(len(ta), len(tb))
    print(f"{nm} producer: issue duration median {np.median(tb[:m] - ta[:m]):7.0f}")
ka = ev[ev[:, 1] == 22, 0].astype(np.int64)
kr = ev[ev[:, 1] == 1, 0].astype(np.int64)
# K tile j issued (ka[j]) -> MMA observed K ready (kr[j])
m = min(len(ka), len(kr))
print("K issued->ready median", np.median(kr[:m] - ka[:m]))

def dur(a, b):
    ta = ev[ev[:, 1] == a, 0].astype(np.int64); tb = ev[ev[:, 1] == b, 0].astype(np.int64)
    m = min(len(ta), len(tb))
    return np.median(tb[:m] - ta[:m]) if m else float("nan")
print("softmax a phases: start->ldS", dur(10, 30), " ldS->max", dur(30, 32), " max->exp", dur(32, 34), " exp->done", dur(34, 12))

# ---- item boundaries (events 40/41: MMA item start / Q ready; 42+h/44+h: epilogue start/end)
def times(c):
    return ev[ev[:, 1] == c, 0].astype(np.int64)
t40, t41 = times(40), times(41)
if len(t41):
    print(f"items {len(t40)}: MMA Q-wait median {np.median(t41 - t40[:len(t41)]):.0f} clk")
    sa = times(7)
    # first S_a issue after each Q ready, and last S_b issue before each item start
    first_sa = np.array([sa[sa > t][0] - t for t in t41 if (sa > t).any()])
    print(f"  Q ready -> first S_a issue median {np.median(first_sa):.0f}")
    span = np.diff(t40)
    print(f"  item period median {np.median(span):.0f} clk, mean {span.mean():.0f}")
for h in (0, 1):
    e0, e1 = times(42 + h), times(44 + h)
    m = min(len(e0), len(e1))
    if m:
        print(f"  epilogue {'ab'[h]} median {np.median(e1[:m] - e0[:m]):.0f} clk")
        st = times(10 + h)
        nxt = np.array([st[st > t][0] - t for t in e1[:m] if (st > t).any()])
        if len(nxt):
            print(f"  epilogue {'ab'[h]} end -> next softmax start median {np.median(nxt):.0f}")
        dn = times(12 + h)
        prev = np.array([t - dn[dn < t][-1] for t in e0[:m] if (dn < t).any()])
        print(f"  last softmax done -> epilogue {'ab'[h]} start (PV wait) median {np.median(prev):.0f}")

for a, w, b, nm in ((20, 24, 22, "K"), (21, 25, 23, "V")):
    ta, tw, tb = times(a), times(w), times(b)
    m = min(len(ta), len(tb), len(tw))
    if m:
        print(f"{nm} (owner warp): empty-wait median {np.median(ta[:m] - tw[:m]):.0f}, issue of 4 sub-blocks median "
              f"{np.median(tb[:m] - ta[:m]):.0f} clk")
kr = times(1)
ki = times(22)
m = min(len(kr), len(ki))
if m:
    print(f"K issue end -> MMA sees K ready median {np.median(kr[:m] - ki[:m]):.0f}")
