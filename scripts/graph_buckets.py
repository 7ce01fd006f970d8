"""NEXT-1 measurement (§6.2, §4.7): eager calls vs CUDA-graph
replay of the batch-size bucket, for config-2-shaped decode batches (32q/8kv, d 128, context
4096, bf16) of B = 1 .. 128 sequences.

  eager        one pattn_unified_attention call with exactly B sequences per step (host
               planning + 3 launches every step)
  graph/exact  replay of the graph recorded for the smallest power-of-two bucket >= B
  graph/128    replay of the 128-sequence bucket's graph holding the same B sequences (the
               paper's "excess instances" of a frozen grid: 128 - B padding sequences, q_b = 0)

Steps rotate over R replicas (different sequences of a 128-sequence, 2.1 GB KV cache) so that
every step misses L2; each graph replica is captured on its own static buffers, filled once
(a server writes its inputs into those buffers directly), so a timed graph step is exactly one
graph launch.  CUDA events, 20 warm-up, mean of 100 steps.  One JSON line per B."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_11581_b200 import pattn  # noqa: E402
from workloads import CONFIGS  # noqa: E402
from workloads.gen import generate_device  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6556.5
w = CONFIGS["c2_decode8b"].with_seqs([(4096, 1)] * 128, name="c2x128")
inp = generate_device(w, seed=5, device="cuda")
kc, vc = inp["k_cache"], inp["v_cache"]
pattn.load()
dev = torch.device("cuda")
s = torch.cuda.Stream(dev)
s2 = torch.cuda.Stream(dev)


def static_set(ids, cap):
    """Static buffers of a `cap`-sequence bucket holding the sequences `ids` (+ padding)."""
    B = len(ids)
    ix = torch.tensor(ids, device=dev)
    b = dict(q=torch.zeros((cap, 32, 128), dtype=torch.bfloat16, device=dev),
             out=torch.zeros((cap, 32, 128), dtype=torch.bfloat16, device=dev),
             bt=torch.zeros((cap, inp["block_table"].shape[1]), dtype=torch.int32, device=dev),
             cu=torch.full((cap + 1,), B, dtype=torch.int32, device=dev),
             sl=torch.zeros(cap, dtype=torch.int32, device=dev))
    b["q"][:B] = inp["q"][ix]
    b["bt"][:B] = inp["block_table"][ix]
    b["cu"][: B + 1] = torch.arange(B + 1, dtype=torch.int32, device=dev)
    b["sl"][:B] = inp["seq_lens"][ix]
    p = pattn.make_problem(b["q"], kc, 8, 16, b["bt"], cap, b["out"], "NHD", 1, 4097)
    b["ws"] = torch.empty(pattn.workspace_size(p), dtype=torch.uint8, device=dev)
    return b


def capture(b):
    return pattn.graph_capture(b["q"], kc, vc, b["bt"], b["cu"], b["sl"], w.scale, 8, 16, b["out"], b["ws"],
                               max_query_len=1, max_seq_len=4097, stream=s, stream2=s2)


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
    R = max(1, min(16, 128 // B))
    sets = [[(r * B + j) % 128 for j in range(B)] for r in range(R)]
    cap = 1 << (B - 1).bit_length()
    exact = [static_set(ids, cap) for ids in sets]
    full = [static_set(ids, 128) for ids in sets]
    g_exact = [capture(b) for b in exact]
    g_full = [capture(b) for b in full]
    torch.cuda.synchronize()

    def eager(i):
        b = exact[i % R]
        pattn.unified_attention(b["q"][:B], kc, vc, b["bt"][:B], b["cu"][: B + 1], b["sl"][:B], w.scale, 8, 16,
                                b["out"][:B], max_query_len=1, max_seq_len=4097, workspace=b["ws"], stream=s,
                                stream2=s2)

    r = {"B": B, "bucket": cap, "replicas": R,
         "eager_us": timeit(eager),
         "graph_exact_us": timeit(lambda i: g_exact[i % R].launch(s)),
         "graph_128_us": timeit(lambda i: g_full[i % R].launch(s))}
    r["launch_saving_us"] = r["eager_us"] - r["graph_exact_us"]
    r["excess_instance_cost_us"] = r["graph_128_us"] - r["graph_exact_us"]
    kv_gb = B * 4097 * 8 * 2 * 128 * 2 / 1e9
    r["graph_exact_hbm_frac"] = kv_gb / (r["graph_exact_us"] * 1e-6) / hbm
    # the replayed outputs agree with the eager ones (bitwise unless the bucket's larger
    # num_seqs lands on another tuning-tree leaf, i.e. another decode segmentation)
    torch.cuda.synchronize()
    eager(0)
    torch.cuda.synchronize()
    ref = exact[0]["out"][:B].float().clone()
    g_full[0].launch(s)
    torch.cuda.synchronize()
    r["graph128_max_abs_diff_vs_eager"] = float((full[0]["out"][:B].float() - ref).abs().max())
    print(json.dumps(r), flush=True)
    for g in g_exact + g_full:
        g.close()
    del exact, full
