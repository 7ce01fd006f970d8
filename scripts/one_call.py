"""One unified_attention call on a device-generated workload (for compute-sanitizer / ncu runs).

  python scripts/one_call.py <workload> [repeat] [seqs_override]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2511_11581_b200 import pattn  # noqa: E402
from workloads import CONFIGS  # noqa: E402
from workloads.gen import generate_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_decode8b"
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = CONFIGS[name]
if len(sys.argv) > 3:  # e.g. "16x4096:1+2x0:300" -> 16 x (ctx 4096, q 1) and 2 x (ctx 0, q 300)
    seqs = []
    for grp in sys.argv[3].split("+"):
        n, rest = grp.split("x")
        ctx, q = rest.split(":")
        seqs += [(int(ctx), int(q))] * int(n)
    w = w.with_seqs(seqs, name=name + "_small")
inp = generate_device(w, seed=1, device="cuda")
out = torch.empty_like(inp["q"])
for _ in range(rep):
    pattn.unified_attention(inp["q"], inp["k_cache"], inp["v_cache"], inp["block_table"], inp["cu_seqlens_q"],
                            inp["seq_lens"], w.scale, w.num_kv_heads, w.block_size, out,
                            max_query_len=max(q for _, q in w.seqs), max_seq_len=max(c + q for c, q in w.seqs))
torch.cuda.synchronize()
print("ok", name, float(out.float().abs().mean()))
