"""NEXT-1 measurement (§6.2, §4.7): eager calls vs CUDA-graph
replay of the batch-size bucket, for config-2-shaped decode batches (32q/8kv, d 128, context
4096, bf16) of B = 1 .. 128 sequences.

  eager        one pattn_unified_attention call with exactly B sequences per step
  graph/exact  replay of the graph recorded for the smallest power-of-two bucket >= B
  graph/128    replay of the 128-sequence bucket for the same B sequences (the "excess
               instances" of a frozen grid: 128 - B padding sequences with q_b = 0)

Steps rotate over 128 different sequences (2.1 GB of KV) so every step misses L2; the per-step
metadata copy into the graph's buffers is inside the timed region.  CUDA events, 20 warm-up,
mean of 100 steps (the paper's protocol).  One JSON line per B on stdout."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_11581_b200 import pattn  # noqa: E402
from paper_2511_11581_b200.graphs import GraphBuckets  # noqa: E402
from workloads import CONFIGS  # noqa: E402
from workloads.gen import generate_device  # noqa: E402

w = CONFIGS["c2_decode8b"].with_seqs([(4096, 1)] * 128, name="c2x128")
inp = generate_device(w, seed=5, device="cuda")
pattn.load()
dev = torch.device("cuda")
gb = GraphBuckets(inp["k_cache"], inp["v_cache"], 32, 8, 16, w.scale, max_query_len=1, max_seq_len=4097)
s = gb.stream
ws = torch.empty(1 << 26, dtype=torch.uint8, device=dev)


def timeit(fn, n=100, warm=20):
    with torch.cuda.stream(s):
        for i in range(warm):
            fn(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(n):
            fn(i)
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for B in (1, 2, 3, 4, 5, 8, 12, 16, 24, 32, 48, 64, 96, 128):
    sets = [torch.arange(r * B, r * B + B, device=dev) % 128 for r in range(max(1, 128 // B))]
    views = [dict(q=inp["q"][ix], bt=inp["block_table"][ix].contiguous(), sl=inp["seq_lens"][ix].contiguous())
             for ix in sets]
    cu = torch.arange(B + 1, dtype=torch.int32, device=dev)
    out = torch.empty((B, 32, 128), dtype=torch.bfloat16, device=dev)

    def eager(i):
        v = views[i % len(views)]
        pattn.unified_attention(v["q"], inp["k_cache"], inp["v_cache"], v["bt"], cu, v["sl"], w.scale, 8, 16, out,
                                max_query_len=1, max_seq_len=4097, workspace=ws, stream=s)

    def graph(bucket):
        def f(i):
            v = views[i % len(views)]
            gb.run(v["q"], v["bt"], cu, v["sl"], bucket=bucket, stream=s)
        return f

    exact = gb.bucket_for(B, B)
    r = {"B": B, "bucket": exact, "eager_us": timeit(eager), "graph_exact_us": timeit(graph(exact)),
         "graph_128_us": timeit(graph(128))}
    r["launch_saving_us"] = r["eager_us"] - r["graph_exact_us"]
    r["excess_instance_cost_us"] = r["graph_128_us"] - r["graph_exact_us"]
    kv_gb = B * 4097 * 8 * 2 * 128 * 2 / 1e9
    r["graph_exact_hbm_frac"] = kv_gb / (r["graph_exact_us"] * 1e-6) / 6556.5
    print(json.dumps(r), flush=True)
gb.close()
