"""K1 load-bound probe: config 3's prefill half (8 x 2048, serial), once with the normal paged
layout and once with every sequence's block table pointing at the SAME physical blocks (K/V of
one sequence, 8 MB, always L2-resident).  Same arithmetic, different K/V memory traffic."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_11581_b200 import pattn  # noqa: E402
from workloads.gen import ATTRIBUTION, generate_device  # noqa: E402

w = ATTRIBUTION["c3p_prefill_part"]
inp = generate_device(w, seed=1, device="cuda")
out = torch.empty_like(inp["q"])
pattn.load()


def run(bt, n=30):
    def call():
        pattn.unified_attention(inp["q"], inp["k_cache"], inp["v_cache"], bt, inp["cu_seqlens_q"], inp["seq_lens"],
                                w.scale, w.num_kv_heads, w.block_size, out, max_query_len=2048, max_seq_len=2048)
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        call()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


flops = w.algorithmic()["flops_prefill"]
t = run(inp["block_table"])
print(f"normal paged KV   : {t:7.1f} us/call  {flops / t / 1e6:7.1f} TFLOP/s")
bt_same = inp["block_table"][0:1].expand_as(inp["block_table"]).contiguous()
t = run(bt_same)
print(f"shared (L2) K/V   : {t:7.1f} us/call  {flops / t / 1e6:7.1f} TFLOP/s")
