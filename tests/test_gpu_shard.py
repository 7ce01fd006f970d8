"""Multi-rank GPU path: world size 2 (gloo; both ranks share GPU 0 here -- NCCL refuses two
ranks on one device, the 8-GPU bench uses NCCL), each rank runs libpattn on its shard of ONE
global batch (by sequence or by KV head, shard.py), the outputs are all-gathered and rank 0
checks the gathered global output against the fp64 oracle element by element and against
the unsharded single-rank libpattn output."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, layout, q_out):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from gpu_helpers import to_torch
        from oracle import attention as O
        from paper_2511_11581_b200 import pattn, shard
        from workloads import Workload, generate

        torch.cuda.set_device(0)
        w = Workload("gpushard", ((0, 300), (2000, 1), (700, 1), (50, 90), (0, 130), (9000, 1), (33, 1), (4000, 1)),
                     32, 8, 128, 16, "bf16")
        b = generate(w, seed=31, dist="peaked", poison=True, layout=layout)
        q, kc, vc = to_torch(b.q), to_torch(b.k_cache), to_torch(b.v_cache)
        plan = shard.plan_shards(b.cu_seqlens_q, b.seq_lens, w.num_q_heads, w.num_kv_heads, w.head_dim, world, mode)
        lb = shard.local_batch(plan, rank, q, kc, vc, b.block_table, b.cu_seqlens_q, b.seq_lens, w.block_size,
                               kv_layout=layout)
        qlens = np.diff(lb.cu_seqlens_q.cpu().numpy())
        local = pattn.unified_attention(lb.q, lb.k_cache, lb.v_cache, lb.block_table, lb.cu_seqlens_q, lb.seq_lens,
                                        w.scale, lb.num_kv_heads, w.block_size, kv_layout=layout,
                                        max_query_len=int(qlens.max()), max_seq_len=int(lb.seq_lens.max().item()))
        torch.cuda.synchronize()
        full = shard.gather_outputs(plan, local.float().cpu(), b.cu_seqlens_q, len(lb.q_heads))  # gloo: fp32
        if rank == 0:
            bt = torch.from_numpy(b.block_table).cuda()
            cu = torch.from_numpy(b.cu_seqlens_q).cuda()
            sl = torch.from_numpy(b.seq_lens).cuda()
            single = pattn.unified_attention(q, kc, vc, bt, cu, sl, w.scale, w.num_kv_heads, w.block_size,
                                             kv_layout=layout, max_query_len=300, max_seq_len=9001)
            torch.cuda.synchronize()
            ref = O.batch_attention(b)
            got = full.double().numpy()
            err = np.abs(got - ref)
            ok = bool(np.isfinite(got).all() and (err <= 1e-2 + 1e-2 * np.abs(ref)).all())
            dsingle = float((full.float() - single.cpu().float()).abs().max())
            q_out.put((ok, float(err.max()), dsingle))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,layout", [("seq", "NHD"), ("kvhead", "NHD"), ("seq", "HND")])
def test_two_rank_libpattn_shards_gather_to_oracle(mode, layout):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, layout, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    ok, err, dsingle = q.get(timeout=10)
    assert ok, f"gathered output out of tolerance: max |err| {err:.3e}"
    assert dsingle <= 2e-2, dsingle
