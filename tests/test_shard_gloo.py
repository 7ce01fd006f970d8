"""Multi-process (world_size 2, gloo, CPU) tests of the batch sharder: each rank builds its
local batch (sequence- or KV-head-sharded), computes its local output (here with the fp64
oracle -- the CUDA kernel needs a GPU), all-gathers, and the gathered global output must equal
the unsharded oracle output bit for bit (rows are independent, so sharding changes nothing)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_11581_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, layout, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import attention as O
        from workloads import Workload, generate

        w = Workload("shard", ((0, 40), (90, 1), (300, 1), (7, 23), (0, 65), (1000, 1), (33, 1)), 8, 2, 64, 16, "f32")
        b = generate(w, seed=21, poison=True, layout=layout)
        plan = shard.plan_shards(b.cu_seqlens_q, b.seq_lens, w.num_q_heads, w.num_kv_heads, w.head_dim, world, mode)
        lb = shard.local_batch(plan, rank, torch.from_numpy(b.q), torch.from_numpy(b.k_cache),
                               torch.from_numpy(b.v_cache), b.block_table, b.cu_seqlens_q, b.seq_lens, w.block_size,
                               kv_layout=layout)
        local = O.paged_attention(lb.q.numpy(), lb.k_cache.numpy(), lb.v_cache.numpy(), lb.block_table.numpy(),
                                  lb.cu_seqlens_q.numpy(), lb.seq_lens.numpy(), w.scale, lb.num_kv_heads,
                                  w.block_size, layout=layout)
        full = shard.gather_outputs(plan, torch.from_numpy(local), b.cu_seqlens_q, len(lb.q_heads) if mode == "seq"
                                    else len(lb.q_heads))
        if rank == 0:
            ref = O.batch_attention(b)
            q_out.put((np.array_equal(full.numpy(), ref), plan.cost.tolist(),
                       [len(x) for x in plan.seq_ids]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,layout", [("seq", "NHD"), ("kvhead", "NHD"), ("seq", "HND"), ("kvhead", "HND")])
def test_shard_gather_roundtrip_world2(mode, layout):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, layout, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    equal, cost, nseq = q.get(timeout=10)
    assert equal
    if mode == "seq":
        assert sum(nseq) == 7 and min(nseq) >= 1


def test_plan_partitions_and_balance():
    rng = np.random.default_rng(0)
    for world in (2, 4, 8):
        qs = np.concatenate([np.full(32, 2048), np.ones(224, np.int64)])
        sl = np.concatenate([np.full(32, 2048), np.full(224, 4097)])
        cu = np.concatenate([[0], np.cumsum(qs)])
        plan = shard.plan_shards(cu, sl, 64, 8, 128, world, "seq")
        allids = np.sort(np.concatenate(plan.seq_ids))
        assert allids.tolist() == list(range(256))
        # config 5's symmetric mix balances exactly: 32/world prefills and 224/world decodes per rank
        for ids in plan.seq_ids:
            assert (qs[ids] > 1).sum() == 32 // world and (qs[ids] == 1).sum() == 224 // world
        assert plan.cost.max() / plan.cost.min() < 1.0001
        # random ragged batch: LPT within (max item) of the mean
        qs = rng.integers(1, 3000, size=97)
        sl = qs + rng.integers(0, 5000, size=97)
        cu = np.concatenate([[0], np.cumsum(qs)])
        plan = shard.plan_shards(cu, sl, 32, 8, 128, world, "seq")
        c = shard.sequence_costs(qs, sl, 32, 8, 128)
        assert plan.cost.max() - plan.cost.min() <= c.max() + 1e-12
    kv = shard.plan_shards(cu, sl, 64, 8, 128, 8, "kvhead")
    assert [list(r) for r in kv.kv_heads] == [[i] for i in range(8)]
    assert kv.q_heads[3] == range(24, 32)


def test_bench_local_workloads_partition_config5():
    # bench.py --shard: every rank's local workload is a disjoint piece of ONE global batch;
    # config 5 at P=8 by sequence = 4 prefills + 28 decodes per rank; by KV head
    # = 1 KV head + 8 query heads per rank over all 256 sequences
    import bench
    from workloads import CONFIGS

    w = CONFIGS["c5_mixed70b"]
    seqs = []
    for r in range(8):
        lw = bench.local_workload(w, "seq", 8, r)
        assert sum(1 for _, q in lw.seqs if q > 1) == 4 and sum(1 for _, q in lw.seqs if q == 1) == 28
        seqs += list(lw.seqs)
    assert sorted(seqs) == sorted(w.seqs)
    for r in range(8):
        lw = bench.local_workload(w, "kvhead", 8, r)
        assert (lw.num_kv_heads, lw.num_q_heads, lw.seqs) == (1, 8, w.seqs)
    assert bench.local_workload(w, "none", 8, 3) is w
