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
         8: "Sb_issued", 10: "SMa_start", 11: "SMb_start", 12: "SMa_done", 13: "SMb_done", 20: "K_load", 21: "V_load"}
print("events", n)
for t, c in ev[:160]:
    print(f"{int(t - t0):8d}  {names.get(int(c), c)}")
# per-event-type mean intervals
for c in sorted(set(ev[:, 1].tolist())):
    ts = ev[ev[:, 1] == c, 0].astype(np.int64)
    if len(ts) > 2:
        d = np.diff(ts)
        print(f"{names.get(c, c):12s} n={len(ts):5d} mean interval {d.mean():8.0f}  median {np.median(d):8.0f}")
sa = ev[ev[:, 1] == 10, 0].astype(np.int64)
da = ev[ev[:, 1] == 12, 0].astype(np.int64)
m = min(len(sa), len(da))
print("softmax a duration median", np.median(da[:m] - sa[:m]))
