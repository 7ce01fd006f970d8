#!/usr/bin/env python
"""bench.py -- libpattn unified paged attention throughput on B200 (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3_mixed8b] [--impl ours|reference]

A "step" is one unified_attention call (one attention layer) over the whole
workload: metadata (K5) + prefill Q blocks (K1/K4) + split-KV decode (K2) + segment
reduce (K3) -- every row of SURVEY.md §8(a).  Default workload: BASELINE.json
config 3 (Llama-3.1-8B shapes, 8 prefills of 2k + 56 decodes at 4k context, bf16),
the configuration that exercises the whole hot path in one unified launch.

N > 1 (torchrun, one process per GPU): each rank processes its own batch of the
same shape (weak scaling; attention shards with no exchange, so there is no
collective on the data path); value = tokens of all ranks / max-over-ranks time.

Timing: W untimed warm-up steps, then EXACTLY K steps bracketed by barrier +
cuda.synchronize, CUDA events on the launching stream; inputs (KV cache >= 1 GB)
are larger than L2, so no flush.  Per-kernel CUDA events (pattn_exec_opts_t.events)
inside the same timed region give each kernel's average duration for the roofline.
SM clocks / throttle reasons are sampled with NVML during the timed region.
`e2e` repeats the measurement through the host-buffer C-ABI call
(pattn_unified_attention_hostio: H2D q+metadata, kernels, D2H out each step).
`cpu_baseline` times the fp64 oracle (oracle/, test infrastructure) on a bounded
random sample of the same workload's tokens on this host's cores (rank 0, N=1).
`--impl reference` times that oracle alone as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "attention tokens/s; decode HBM GB/s & prefill TFLOP/s vs B200 peak, 1/2/4/8 GPUs"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="c3_mixed8b")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--streams", type=int, default=2,
                    help="2 (default): decode kernels on a second stream, concurrent with prefill; 1: serial")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--seed", type=int, default=3003)
    ap.add_argument("--shard", default="none", choices=["none", "seq", "kvhead"],
                    help="N>1: split ONE global batch of the workload over the ranks (strong scaling; "
                         "shard.py plan); none = every rank runs the full workload (weak scaling)")
    ap.add_argument("--sim-world", type=int, default=0,
                    help="with --shard: run rank --sim-rank of a --sim-world-way shard on this one GPU")
    ap.add_argument("--sim-rank", type=int, default=0)
    return ap.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sustained=d.get("bf16_tflops_sustained"),
                    sm_max=d.get("sm_max_mhz"), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sustained=1400.0, sm_max=1965.0, src="fallback")


# ----------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    """Polls SM clock and clock-event reasons every ~5 ms while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": names,
            "samples": len(self.samples),
        }


# ----------------------------------------------------------------------------- work accounting
def kernel_work(w):
    """Algorithmic work per step: causally visible (row,key) pairs
    only; KV bytes read once per (sequence, KV head)."""
    a = w.algorithmic()
    D, Hq, esz = w.head_dim, w.num_q_heads, 2 if w.dtype == "bf16" else 4
    n_dec = sum(1 for _, q in w.seqs if q == 1)
    n_pre_tok = sum(q for _, q in w.seqs if q > 1)
    return dict(
        prefill_flops=a["flops_prefill"],
        decode_bytes=a["bytes_kv_decode"] + 2.0 * n_dec * Hq * D * esz,  # KV + q + out of decode tokens
        prefill_bytes=a["bytes_kv_prefill"] + 2.0 * n_pre_tok * Hq * D * esz,
        total_flops=a["flops"],
        total_bytes=a["bytes"],
    )


# ----------------------------------------------------------------------------- oracle sample
def oracle_sample(w, host, n_tokens, rng, threads):
    """Time the fp64 oracle on n_tokens random query tokens (all heads) of the workload."""
    from oracle import attention as O

    T = w.num_tokens
    toks = np.sort(rng.choice(T, size=min(n_tokens, T), replace=False))
    rows = (toks[:, None] * w.num_q_heads + np.arange(w.num_q_heads)[None, :]).reshape(-1)
    t0 = time.perf_counter()
    O.paged_attention(host["q"], host["k"], host["v"], host["bt"], host["cu"], host["sl"], w.scale,
                      w.num_kv_heads, w.block_size, layout=host["layout"], rows=rows, threads=threads)
    return time.perf_counter() - t0, len(toks)


def host_inputs_from_device(inp):
    import torch

    def bits(t):
        return t.view(torch.int16).cpu().numpy().view(np.uint16) if t.dtype == torch.bfloat16 else t.cpu().numpy()

    from oracle import attention as O

    return dict(
        q=O.widen(bits(inp["q"])), k=O.widen(bits(inp["k_cache"])), v=O.widen(bits(inp["v_cache"])),
        bt=inp["block_table_h"].numpy(), cu=inp["cu_seqlens_q_h"].numpy(), sl=inp["seq_lens_h"].numpy(),
        layout=inp["layout"],
    )


def cpu_baseline(w, inp, target_s=12.0):
    from oracle import attention as O

    cores = len(os.sched_getaffinity(0))
    host = host_inputs_from_device(inp)
    rng = np.random.default_rng(7)
    oracle_sample(w, host, 8, rng, cores)  # first touch of the widened host arrays
    t_cal, n_cal = oracle_sample(w, host, 32, rng, cores)
    n = max(8, min(w.num_tokens, int(n_cal * target_s / max(t_cal, 1e-3))))
    t, n = oracle_sample(w, host, n, rng, cores)
    return {
        "value": n / t,
        "unit": "tokens/s",
        "cores": int(O.max_threads() if cores <= 0 else cores),
        "kind": "oracle",
        "sample": f"{n} of {w.num_tokens} query tokens drawn uniformly at random (all {w.num_q_heads} heads), "
                  f"fp64 C/OpenMP oracle, {t:.1f} s",
    }


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from workloads import CONFIGS, generate
    from oracle import attention as O

    w = CONFIGS[args.workload]
    b = generate(w, seed=args.seed, poison=False)
    host = dict(q=O.widen(b.q), k=O.widen(b.k_cache), v=O.widen(b.v_cache), bt=b.block_table, cu=b.cu_seqlens_q,
                sl=b.seq_lens, layout=b.layout)
    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(11)
    oracle_sample(w, host, 64, rng, cores)  # first touch of the widened host arrays
    t_cal, n_cal = oracle_sample(w, host, 64, rng, cores)
    per_step = max(1, min(w.num_tokens, int(n_cal * 0.25 / max(t_cal, 1e-4))))
    for _ in range(args.warmup):
        oracle_sample(w, host, per_step, rng, cores)
    tot_t, tot_n = 0.0, 0
    for _ in range(args.steps):
        t, n = oracle_sample(w, host, per_step, rng, cores)
        tot_t += t
        tot_n += n
    value = tot_n / tot_t
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if args.shard == "none" else "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.workload, "tokens_per_step": per_step,
                   "note": "fp64 CPU oracle on a random sample of the workload's query tokens per step"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": f"{per_step} random query tokens (all heads) per step"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2511_11581_b200 import pattn
    from workloads import CONFIGS
    from workloads.gen import ATTRIBUTION, generate_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PATTN_BENCH_BACKEND=gloo: test-only oversubscription (several ranks sharing one GPU, which
    # NCCL refuses) to exercise the multi-rank path on a 1-GPU box; never used for numbers
    backend = os.environ.get("PATTN_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    pattn.load()

    w_global = CONFIGS[args.workload] if args.workload in CONFIGS else ATTRIBUTION[args.workload]
    shard_world = args.sim_world if args.sim_world else world
    shard_rank = args.sim_rank if args.sim_world else rank
    w = local_workload(w_global, args.shard, shard_world, shard_rank)
    inp = generate_device(w, seed=args.seed + rank, device=dev)
    q, kc, vc = inp["q"], inp["k_cache"], inp["v_cache"]
    bt, cu, sl = inp["block_table"], inp["cu_seqlens_q"], inp["seq_lens"]
    out = torch.empty_like(q)
    max_q = max(qq for _, qq in w.seqs)
    max_L = max(c + qq for c, qq in w.seqs)
    prob = pattn.make_problem(q, kc, w.num_kv_heads, w.block_size, bt, w.num_seqs, out, "NHD", max_q, max_L,
                              args.flags)
    launches_per_step = pattn.planned_launches(prob)
    stream = torch.cuda.current_stream(dev)
    stream2 = torch.cuda.Stream(dev) if args.streams == 2 else None

    def step(events=None):
        pattn.unified_attention(q, kc, vc, bt, cu, sl, w.scale, w.num_kv_heads, w.block_size, out,
                                max_query_len=max_q, max_seq_len=max_L, flags=args.flags, stream=stream,
                                stream2=stream2, events=events)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    K = args.steps
    NK = pattn.KERNEL_COUNT
    kmask = pattn.planned_kernels(prob)
    kev = pattn.make_events(K)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        t0.record(stream)
        for i in range(K):
            step(kev[i])
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = t0.elapsed_time(t1) / K
    # K1's SM share in the timed steps (K5's two-stream partition; all SMs when serial)
    prefill_sms_timed = pattn.last_prefill_sms(local)
    # per-kernel average durations (only kinds that were launched)
    kern_ms = {}
    for k in range(NK):
        if kmask & (1 << k):
            kern_ms[pattn.KERNEL_NAMES[k]] = sum(kev[i][2 * k].elapsed_time(kev[i][2 * k + 1]) for i in range(K)) / K

    if args.shard == "none":
        tokens_all = w.num_tokens * world  # weak scaling: every rank runs the full workload
    elif args.sim_world:
        tokens_all = w.num_tokens if args.shard == "seq" else w.num_tokens / args.sim_world  # this rank's share
    else:
        tokens_all = w_global.num_tokens  # strong scaling: one global batch split over the ranks

    # ---------------- the same step captured once as a CUDA graph and replayed (static grids,
    # device-resident metadata: P:190-199); reported beside the eager number
    graph = None
    try:
        gs = torch.cuda.Stream(dev)
        gs2 = torch.cuda.Stream(dev) if args.streams == 2 else None
        with torch.cuda.stream(gs):
            pattn.unified_attention(q, kc, vc, bt, cu, sl, w.scale, w.num_kv_heads, w.block_size, out,
                                    max_query_len=max_q, max_seq_len=max_L, flags=args.flags, stream=gs,
                                    stream2=gs2)
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, stream=gs):
            pattn.unified_attention(q, kc, vc, bt, cu, sl, w.scale, w.num_kv_heads, w.block_size, out,
                                    max_query_len=max_q, max_seq_len=max_L, flags=args.flags, stream=gs,
                                    stream2=gs2)
        for _ in range(3):
            cg.replay()
        torch.cuda.synchronize()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        rs = torch.cuda.current_stream(dev)  # CUDAGraph.replay() launches on the current stream
        g0.record(rs)
        for _ in range(K):
            cg.replay()
        g1.record(rs)
        torch.cuda.synchronize()
        gms = torch.tensor([g0.elapsed_time(g1) / K], device=dev)
        if world > 1:
            dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        ref_out = out.clone()
        out.fill_(0)
        cg.replay()
        torch.cuda.synchronize()
        same = bool(torch.equal(out, ref_out))
        graph = {"ms_per_step": float(gms.item()), "value": tokens_all / (float(gms.item()) * 1e-3),
                 "replay_matches_eager": same}
    except Exception as ex:  # reported, never fatal
        graph = {"error": str(ex)[:200]}

    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = tokens_all / (ms_max * 1e-3)

    # ---------------- e2e through the host-buffer C-ABI call.  Steps alternate between two
    # streams with their own workspaces and pinned output buffers (a server keeping two
    # requests in flight): step i+1's H2D overlaps step i's kernels and D2H (PCIe is full
    # duplex).  Every step still copies its whole q + metadata in and its whole out back.
    e2e = None
    if not args.no_e2e:
        q_h = q.cpu().pin_memory()
        outs_h = [torch.empty_like(q_h).pin_memory() for _ in range(2)]
        out_h = outs_h[0]
        bt_h, cu_h, sl_h = (inp["block_table_h"].pin_memory(), inp["cu_seqlens_q_h"].pin_memory(),
                            inp["seq_lens_h"].pin_memory())
        hp = pattn.make_problem(q_h, kc, w.num_kv_heads, w.block_size, bt_h, w.num_seqs, out_h, "NHD", max_q, max_L,
                                args.flags)
        hws = [torch.empty(pattn.hostio_workspace_size(hp), dtype=torch.uint8, device=dev) for _ in range(2)]
        hst = [stream, torch.cuda.Stream(dev)]

        def step_h(i):
            pattn.unified_attention_hostio(q_h, kc, vc, bt_h, cu_h, sl_h, w.scale, w.num_kv_heads, w.block_size,
                                           outs_h[i % 2], max_query_len=max_q, max_seq_len=max_L, flags=args.flags,
                                           workspace=hws[i % 2], stream=hst[i % 2])

        for i in range(4):
            step_h(i)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        hst[1].wait_stream(stream)
        for i in range(K):
            step_h(i)
        stream.wait_stream(hst[1])
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1) / K], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        esz = q.element_size()
        h2d = q_h.numel() * esz + bt_h.numel() * 4 + cu_h.numel() * 4 + sl_h.numel() * 4
        d2h = out_h.numel() * esz
        e2e = {"value": tokens_all / (float(ems.item()) * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": float(ems.item()), "requests_in_flight": 2}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks = load_peaks()
    work = kernel_work(w)
    num_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    prefill_sms = prefill_sms_timed if pre_sms_known(kmask, pattn) else num_sms
    sm_share = min(1.0, prefill_sms / num_sms)
    rl = {}
    pre_name = "prefill" if "prefill" in kern_ms else ("generic" if "generic" in kern_ms else None)
    traffic = load_traffic(args.workload)
    if pre_name and work["prefill_flops"] > 0:
        t = kern_ms[pre_name] * 1e-3
        a = work["prefill_flops"] / t / 1e12
        # two streams: K1 runs on the P SMs K5 gave it (the decode kernel has the rest), so its
        # tensor roof is the measured peak x P / #SMs; serial: P = all SMs
        pk = peaks["bf16"] * sm_share
        rl["prefill"] = {"bound": "tensor", "achieved": a, "peak": pk, "unit": "TFLOP/s",
                         "frac": a / pk, "traffic": traffic.get(pre_name), "kernel": pre_name,
                         "kernel_ms": kern_ms[pre_name], "share_of_step": kern_ms[pre_name] / ms,
                         "prefill_sms": prefill_sms, "num_sms": num_sms}
    if "decode" in kern_ms and work["decode_bytes"] > 0:
        t = kern_ms["decode"] * 1e-3
        a = work["decode_bytes"] / t / 1e9
        rl["decode"] = {"bound": "hbm", "achieved": a, "peak": peaks["hbm"], "unit": "GB/s",
                        "frac": a / peaks["hbm"], "traffic": traffic.get("decode"), "kernel": "decode",
                        "kernel_ms": kern_ms["decode"], "share_of_step": kern_ms["decode"] / ms}
    if "baseline" in kern_ms:  # the paper's App. A kernel (--flags 16): SIMT, reported by time only
        rl["baseline"] = {"bound": "alu", "achieved": work["total_flops"] / (kern_ms["baseline"] * 1e-3) / 1e12,
                          "peak": None, "unit": "TFLOP/s", "frac": None, "traffic": None, "kernel": "baseline",
                          "kernel_ms": kern_ms["baseline"], "share_of_step": kern_ms["baseline"] / ms}
    dominant = max(rl.values(), key=lambda r: r["kernel_ms"]) if rl else None

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline(w, inp)
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "tokens/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                   "sample": f"failed: {ex}"}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": K,
        "warmup": max(3, args.warmup),
        "ms_per_step": ms_max,
        "higher_is_better": True,
        "scaling": "weak" if args.shard == "none" else "strong",
        "vs_baseline": None,
        "dtype": "bf16" if w.dtype == "bf16" else "f32",
        "data": "synthetic",
        "config": {
            "workload": args.workload,
            "seqs": f"{sum(1 for _, q in w.seqs if q > 1)} prefill x {max_q} tok + "
                    f"{sum(1 for _, q in w.seqs if q == 1)} decode @ ctx {max((c for c, q in w.seqs if q == 1), default=0)}",
            "heads": f"{w.num_q_heads}q/{w.num_kv_heads}kv x d{w.head_dim}",
            "block_size": w.block_size,
            "tokens_per_step_per_gpu": w.num_tokens,
            "parallelism": parallelism_text(args, world, w_global, w),
            **({"comm_backend_test_only": backend} if backend != "nccl" else {}),
            "l2": "inputs > L2 (KV cache %.2f GB/GPU), no flush" % (kc.numel() * 2 * kc.element_size() / 1e9),
            "streams": args.streams,
            "flags": args.flags,
            "peaks": peaks["src"],
        },
        "roofline": ({k: dominant[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}
                     if dominant else None),
        "roofline_kernels": rl,
        "kernel_ms": kern_ms,
        "clocks": sampler.summary(),
        "e2e": e2e,
        "cuda_graph": graph,
        "gpu_launches": launches_per_step * K,
        "cpu_baseline": cpu,
        "algorithmic": {"prefill_tflop_per_step": work["prefill_flops"] / 1e12,
                        "decode_gb_per_step": work["decode_bytes"] / 1e9,
                        "step_tflops": work["total_flops"] / (ms * 1e-3) / 1e12,
                        "step_gbs": work["total_bytes"] / (ms * 1e-3) / 1e9},
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def pre_sms_known(kmask, pattn):
    return bool(kmask & (1 << pattn.KERNEL_PREFILL))


def local_workload(w, mode, world, rank):
    """This rank's share of ONE global batch (shard.py plan).  Mode "seq": the
    rank's sequences (class-aware LPT balance); "kvhead": the rank's Hkv/P KV heads and their
    query heads for every sequence.  Mode "none" or world 1: the workload itself."""
    if mode == "none" or world <= 1:
        return w
    from paper_2511_11581_b200 import shard

    q_lens = np.array([q for _, q in w.seqs], np.int64)
    cu = np.concatenate([[0], np.cumsum(q_lens)])
    sl = np.array([c + q for c, q in w.seqs], np.int64)
    plan = shard.plan_shards(cu, sl, w.num_q_heads, w.num_kv_heads, w.head_dim, world, mode)
    if mode == "kvhead":
        return w.__class__(f"{w.name}/kvhead{rank}of{world}", w.seqs, len(plan.q_heads[rank]),
                           len(plan.kv_heads[rank]), w.head_dim, w.block_size, w.dtype)
    return w.with_seqs([w.seqs[b] for b in plan.seq_ids[rank]], name=f"{w.name}/seq{rank}of{world}")


def parallelism_text(args, world, w_global, w):
    if args.shard == "none":
        return f"dp{world} (every rank runs the full workload; no collective)"
    if args.sim_world:
        return (f"{args.shard}-shard rank {args.sim_rank} of {args.sim_world} run alone on 1 GPU "
                f"({w.num_seqs} seqs, {w.num_q_heads}q/{w.num_kv_heads}kv heads; value = this rank's tokens/s)")
    return f"{args.shard}-sharded global batch over {world} ranks (strong scaling; no collective)"


def load_traffic(workload):
    """ncu dram bytes per launch, from the committed profile summary of this round (or {})."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        try:
            return json.load(open(path)).get(workload, {})
        except Exception:
            return {}
    return {}


if __name__ == "__main__":
    sys.exit(main())
