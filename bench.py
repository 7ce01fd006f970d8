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
    ap.add_argument("--no-sub", action="store_true", help="skip the keyed sub-results (other configs)")
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
    D, Hq, esz = w.head_dim, w.num_q_heads, 4 if w.dtype == "f32" else 2
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


def cpu_baseline(w, seed, dev, target_s=12.0):
    """The fp64 oracle on this host's cores, on the same inputs (regenerated from the seed)."""
    from oracle import attention as O
    from workloads.gen import generate_device

    cores = len(os.sched_getaffinity(0))
    host = host_inputs_from_device(generate_device(w, seed=seed, device=dev))
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
class Case:
    """One workload resident on the device (inputs > L2, or rotated replicas of it) plus the
    unified call over it.  `step(i)` enqueues call i (replica i mod R)."""

    def __init__(self, w, seed, dev, pattn, streams, flags, l2_bytes, inp=None):
        import torch

        from workloads.gen import generate_device

        self.w, self.dev, self.pattn, self.flags = w, dev, pattn, flags
        first = inp if inp is not None else generate_device(w, seed=seed, device=dev)
        ws_bytes = sum(first[k].numel() * first[k].element_size() for k in ("q", "k_cache", "v_cache"))
        # working set below 2 x L2: rotate R input replicas so every call misses L2
        self.replicas = 1 if ws_bytes >= 2 * l2_bytes else int(math.ceil(2 * l2_bytes / max(ws_bytes, 1)))
        self.inps = [first] + [generate_device(w, seed=seed + 7919 * r, device=dev) for r in range(1, self.replicas)]
        self.ws_bytes = ws_bytes
        self.outs = [torch.empty_like(i["q"]) for i in self.inps]
        self.max_q = max(qq for _, qq in w.seqs)
        self.max_L = max(c + qq for c, qq in w.seqs)
        i0 = self.inps[0]
        self.prob = pattn.make_problem(i0["q"], i0["k_cache"], w.num_kv_heads, w.block_size, i0["block_table"],
                                       w.num_seqs, self.outs[0], "NHD", self.max_q, self.max_L, flags)
        self.stream = torch.cuda.current_stream(dev)
        self.stream2 = torch.cuda.Stream(dev) if streams == 2 else None
        self.streams = streams
        nbytes = pattn.workspace_size(self.prob)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)

    @property
    def out(self):
        return self.outs[0]

    def step(self, i=0, events=None, stream=None, stream2=None):
        r = i % self.replicas
        x, w = self.inps[r], self.w
        self.pattn.unified_attention(
            x["q"], x["k_cache"], x["v_cache"], x["block_table"], x["cu_seqlens_q"], x["seq_lens"], w.scale,
            w.num_kv_heads, w.block_size, self.outs[r], max_query_len=self.max_q, max_seq_len=self.max_L,
            flags=self.flags, workspace=self.workspace, stream=stream or self.stream,
            stream2=stream2 if stream is not None else self.stream2, events=events)

    def prefill_sms(self):
        return self.pattn.workspace_prefill_sms(self.workspace)


def timed(case, K, W, barrier, with_events=True):
    """W untimed calls, then K calls between CUDA events on the launching stream (barrier +
    synchronize on both sides): the step time.  With `with_events`, a second timed region of K
    calls follows in which the library records CUDA events around every kernel
    (pattn_exec_opts_t.events) -- the per-kernel averages for the roofline.  The two are
    separate because those per-kernel event records are not free: they add ~2 us between
    kernels (config 2: 177 us per call plain vs 193 us instrumented), so the step time is
    measured without them.  Returns (ms_per_step, kernel_ms, instrumented_ms_per_step)."""
    import torch

    pattn = case.pattn
    for i in range(max(3, W)):
        case.step(i)
    torch.cuda.synchronize()

    def region(kev):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        t0.record(case.stream)
        for i in range(K):
            case.step(i, events=kev[i] if kev else None)
        t1.record(case.stream)
        torch.cuda.synchronize()
        barrier()
        return t0.elapsed_time(t1) / K

    ms = region(None)
    kern_ms, ms_instr = {}, None
    if with_events:
        kev = pattn.make_events(K)
        # the two regions are separate measurements: let the clocks recover from the first
        # (a long tensor-core burst can drop the SM clock) and warm up again before the second
        time.sleep(0.5)
        for i in range(3):
            case.step(i)
        torch.cuda.synchronize()
        ms_instr = region(kev)
        kmask = pattn.planned_kernels(case.prob)
        for k in range(pattn.KERNEL_COUNT):
            if kmask & (1 << k):
                kern_ms[pattn.KERNEL_NAMES[k]] = sum(kev[i][2 * k].elapsed_time(kev[i][2 * k + 1])
                                                     for i in range(K)) / K
    return ms, kern_ms, ms_instr


def fp32_fma_peak_tflops(num_sms, peaks):
    """SIMT fp32 roof for the generic kernel K4: 128 FP32 lanes x 2 flop (FFMA) per SM per clock at
    the maximum SM clock (B200_PROFILING.md unit counts; 148 SMs x 128 x 2 x 1.965 GHz = 74.4)."""
    return num_sms * 128 * 2 * (peaks.get("sm_max") or 1965.0) * 1e6 / 1e12


def roofline_of(case, ms, kern_ms, peaks, num_sms, traffic):
    """Per-kernel roofline entries: algorithmic work / the kernel's average event time / the
    FULL measured peak of the GPU (MEASURED_PEAKS.json).  With two streams K1 runs on the P SMs
    K5 gave it; the fraction of that share's roof is reported separately (`frac_of_sm_share`).
    `ideal_ms` = work / peak orders the kernels: the one with the largest is the step's
    dominant roof (concurrent kernels can share the same event span)."""
    work = kernel_work(case.w)
    rl = {}
    pre_name = "prefill" if "prefill" in kern_ms else ("generic" if "generic" in kern_ms else None)
    if pre_name and work["prefill_flops"] > 0:
        t = kern_ms[pre_name] * 1e-3
        a = work["prefill_flops"] / t / 1e12
        if pre_name == "prefill":
            bound, pk = "tensor", peaks["bf16"]
        else:  # SIMT fallback / fp32 path
            bound, pk = "alu", fp32_fma_peak_tflops(num_sms, peaks)
        e = {"bound": bound, "achieved": a, "peak": pk, "unit": "TFLOP/s", "frac": a / pk,
             "traffic": traffic.get(pre_name), "kernel": pre_name, "kernel_ms": kern_ms[pre_name],
             "share_of_step": kern_ms[pre_name] / ms, "ideal_ms": work["prefill_flops"] / (pk * 1e12) * 1e3,
             "algorithmic_unit": "4*D*Hq*(ctx_b+i+1) flop per prefill query token (visible pairs only)"}
        if pre_name == "prefill" and case.streams == 2 and "decode" in kern_ms:
            sms = case.prefill_sms()
            e["prefill_sms"] = sms
            e["frac_of_sm_share"] = a / (pk * sms / num_sms)
        rl["prefill"] = e
    dec_name = "decode" if "decode" in kern_ms else ("generic" if "generic" in kern_ms else None)
    if dec_name and work["decode_bytes"] > 0:
        t = kern_ms[dec_name] * 1e-3
        a = work["decode_bytes"] / t / 1e9
        rl["decode"] = {"bound": "hbm", "achieved": a, "peak": peaks["hbm"], "unit": "GB/s", "frac": a / peaks["hbm"],
                        "traffic": traffic.get(dec_name), "kernel": dec_name, "kernel_ms": kern_ms[dec_name],
                        "share_of_step": kern_ms[dec_name] / ms,
                        "ideal_ms": work["decode_bytes"] / (peaks["hbm"] * 1e9) * 1e3,
                        "algorithmic_unit": "L_b*Hkv*2*D*esz B of K+V + 2*Hq*D*esz B of q/out per decode sequence"}
    if "baseline" in kern_ms:  # the paper's App. A kernel (--flags 16): SIMT, reported by time only
        rl["baseline"] = {"bound": "alu", "achieved": work["total_flops"] / (kern_ms["baseline"] * 1e-3) / 1e12,
                          "peak": None, "unit": "TFLOP/s", "frac": None, "traffic": None, "kernel": "baseline",
                          "kernel_ms": kern_ms["baseline"], "share_of_step": kern_ms["baseline"] / ms,
                          "ideal_ms": 0.0}
    return rl


def dominant_roof(rl):
    return max(rl.values(), key=lambda r: (r["ideal_ms"], r["kernel_ms"])) if rl else None


def sub_result(name, w, dev, pattn, streams, K, W, peaks, num_sms, l2, barrier, seed):
    """A second workload timed in the same run (keyed sub-result of the JSON line)."""
    import torch

    case = Case(w, seed, dev, pattn, streams, 0, l2)
    ms, kern_ms, ms_instr = timed(case, K, W, barrier)
    rl = roofline_of(case, ms_instr, kern_ms, peaks, num_sms, load_traffic(name))
    dom = dominant_roof(rl)
    r = {"workload": name, "streams": streams, "ms_per_step": ms, "value": w.num_tokens / (ms * 1e-3),
         "unit": "tokens/s", "kernel_ms": kern_ms, "instrumented_ms_per_step": ms_instr, "replicas": case.replicas,
         "l2": "inputs %.2f GB %s" % (case.ws_bytes / 1e9, "> 2x L2, no flush" if case.replicas == 1 else
                                      f"< 2x L2: {case.replicas} rotated replicas"),
         "roofline": ({k: dom[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "kernel")}
                      if dom else None)}
    del case
    torch.cuda.empty_cache()
    return r


def strong_scaling_c5(args, dev, pattn, world, rank, barrier, l2):
    """Config 5 (256 sequences, 70B heads) as ONE global batch split over the ranks by sequence
    and by KV head (shard.py; no collective on the timed path).  Each rank generates the same
    global batch (same seed), builds its shard, and the shards are timed together (max over
    ranks).  Verification (untimed): the shards' outputs are all-gathered over NCCL and rank 0
    compares them with its own unsharded single-GPU output of the global batch."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_11581_b200 import shard
    from workloads import CONFIGS
    from workloads.gen import generate_device

    w = CONFIGS["c5_mixed70b"]
    K = min(args.steps, 50)
    g = generate_device(w, seed=args.seed + 555, device=dev)
    res = {"workload": "c5_mixed70b", "global_tokens": w.num_tokens}
    # P = 1 point of the curve: the whole batch on this GPU (rank 0; the others wait)
    ref = None
    if rank == 0:
        full = Case(w, 0, dev, pattn, 2, 0, l2, inp=g)
        ms1, _, _ = timed(full, K, args.warmup, lambda: None, with_events=False)
        ref = full.out.clone()
        res["one_gpu_ms"] = ms1
        del full
    barrier()
    if world == 1:
        res["value_one_gpu"] = w.num_tokens / (res["one_gpu_ms"] * 1e-3)
        return res
    cu_h, sl_h, bt_h = g["cu_seqlens_q_h"].numpy(), g["seq_lens_h"].numpy(), g["block_table_h"].numpy()
    for mode in ("seq", "kvhead"):
        plan = shard.plan_shards(cu_h, sl_h, w.num_q_heads, w.num_kv_heads, w.head_dim, world, mode)
        lb = shard.local_batch(plan, rank, g["q"], g["k_cache"], g["v_cache"], bt_h, cu_h, sl_h, w.block_size, dev)
        if mode == "kvhead":
            lw = w.__class__(f"c5/kvhead{rank}of{world}", w.seqs, len(lb.q_heads), lb.num_kv_heads, w.head_dim,
                             w.block_size, w.dtype)
        else:
            lw = w.with_seqs([w.seqs[b] for b in plan.seq_ids[rank]], name=f"c5/seq{rank}of{world}")
        linp = dict(q=lb.q, k_cache=lb.k_cache, v_cache=lb.v_cache, block_table=lb.block_table,
                    cu_seqlens_q=lb.cu_seqlens_q, seq_lens=lb.seq_lens)
        case = Case(lw, 0, dev, pattn, 2, 0, l2, inp=linp)
        ms, _, _ = timed(case, K, args.warmup, barrier, with_events=False)
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
        if dist.get_backend() == "gloo":  # test-only multi-rank runs on one GPU: gather on the host
            gathered = shard.gather_outputs(plan, case.out.cpu(), cu_h, w.num_q_heads).to(dev)
        else:  # NCCL over NVLink
            gathered = shard.gather_outputs(plan, case.out, cu_h, w.num_q_heads)
        entry = {"ms_per_step": ms_max, "value": w.num_tokens / (ms_max * 1e-3), "unit": "tokens/s",
                 "local_seqs": int(lw.num_seqs), "local_heads": f"{lw.num_q_heads}q/{lw.num_kv_heads}kv",
                 "replicas": case.replicas}
        if rank == 0:
            rng = np.random.default_rng(5)
            rows = torch.from_numpy(np.sort(rng.choice(w.num_tokens, size=min(4096, w.num_tokens), replace=False)))
            rows = rows.to(dev)
            a, b = gathered.index_select(0, rows).float(), ref.index_select(0, rows).float()
            diff = (a - b).abs()
            entry["verify"] = {
                "rows_sampled": int(rows.numel()),
                "bitwise_equal": bool(torch.equal(gathered.index_select(0, rows), ref.index_select(0, rows))),
                "max_abs_diff_vs_unsharded": float(diff.max().item()),
                # plans differ per shard (K5 sizes decode segments from the local batch), so the
                # outputs agree to the bf16 tolerance rather than bitwise in general
                "within_bf16_tol": bool((diff <= 1e-2 + 1e-2 * b.abs()).all().item()),
            }
            entry["efficiency_vs_one_gpu"] = res["one_gpu_ms"] / (world * ms_max)
        res[mode] = entry
        del case, lb, linp, gathered
        torch.cuda.empty_cache()
        barrier()
    if rank == 0:
        res["verified"] = all(res[m]["verify"]["within_bf16_tol"] for m in ("seq", "kvhead"))
    return res


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2511_11581_b200 import pattn
    from workloads import CONFIGS
    from workloads.gen import ATTRIBUTION

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
    props = torch.cuda.get_device_properties(dev)
    num_sms = props.multi_processor_count
    l2 = int(getattr(props, "L2_cache_size", 126 << 20) or (126 << 20))
    peaks = load_peaks()

    def barrier():
        if world > 1:
            dist.barrier()

    w_global = CONFIGS[args.workload] if args.workload in CONFIGS else ATTRIBUTION[args.workload]  # + envelope shapes
    shard_world = args.sim_world if args.sim_world else world
    shard_rank = args.sim_rank if args.sim_world else rank
    w = local_workload(w_global, args.shard, shard_world, shard_rank)
    case = Case(w, args.seed + rank, dev, pattn, args.streams, args.flags, l2)
    inp = case.inps[0]
    q, kc = inp["q"], inp["k_cache"]
    launches_per_step = pattn.planned_launches(case.prob)
    K = args.steps

    sampler = ClockSampler(local)
    with sampler:
        ms, kern_ms, ms_instr = timed(case, K, args.warmup, barrier)

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
            case.step(0, stream=gs, stream2=gs2)
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, stream=gs):
            case.step(0, stream=gs, stream2=gs2)
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
        ref_out = case.out.clone()
        case.out.fill_(0)
        cg.replay()
        torch.cuda.synchronize()
        same = bool(torch.equal(case.out, ref_out))
        graph = {"ms_per_step": float(gms.item()), "value": tokens_all / (float(gms.item()) * 1e-3),
                 "replay_matches_eager": same,
                 "note": "replicas not rotated (one captured call)" if case.replicas > 1 else None}
        del cg
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
        vc = inp["v_cache"]
        q_h = q.cpu().pin_memory()
        outs_h = [torch.empty_like(q_h).pin_memory() for _ in range(2)]
        out_h = outs_h[0]
        bt_h, cu_h, sl_h = (inp["block_table_h"].pin_memory(), inp["cu_seqlens_q_h"].pin_memory(),
                            inp["seq_lens_h"].pin_memory())
        hp = pattn.make_problem(q_h, kc, w.num_kv_heads, w.block_size, bt_h, w.num_seqs, out_h, "NHD", case.max_q,
                                case.max_L, args.flags)
        hws = [torch.empty(pattn.hostio_workspace_size(hp), dtype=torch.uint8, device=dev) for _ in range(2)]
        hst = [case.stream, torch.cuda.Stream(dev)]

        def step_h(i):
            pattn.unified_attention_hostio(q_h, kc, vc, bt_h, cu_h, sl_h, w.scale, w.num_kv_heads, w.block_size,
                                           outs_h[i % 2], max_query_len=case.max_q, max_seq_len=case.max_L,
                                           flags=args.flags, workspace=hws[i % 2], stream=hst[i % 2])

        for i in range(4):
            step_h(i)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(case.stream)
        hst[1].wait_stream(case.stream)
        for i in range(K):
            step_h(i)
        case.stream.wait_stream(hst[1])
        e1.record(case.stream)
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
        del q_h, outs_h, hws

    rl = roofline_of(case, ms_instr, kern_ms, peaks, num_sms, load_traffic(args.workload))
    dominant = dominant_roof(rl)
    kv_gb = kc.numel() * 2 * kc.element_size() / 1e9
    work = kernel_work(w)
    del case, inp, q, kc
    torch.cuda.empty_cache()

    # ---------------- keyed sub-results measured in the same run (north_star targets): config-4
    # long-context decode and config-2 decode (K2 vs HBM), K1 alone on config 3's prefill half
    # (serial, whole GPU, vs bf16), and config 5 as one global batch: on 1 GPU at N = 1, split
    # by sequence and by KV head over the ranks (strong scaling, verified) at N > 1
    subs = {}
    if not args.no_sub and args.shard == "none" and not args.sim_world:
        if world == 1:
            Ks = min(K, 50)
            for name, wl, st in (("c4_decode128k", CONFIGS["c4_decode128k"], 1),
                                 ("c2_decode8b", CONFIGS["c2_decode8b"], 1),
                                 ("c3p_prefill_part", ATTRIBUTION["c3p_prefill_part"], 1)):
                if name == args.workload:
                    continue
                try:
                    subs[name] = sub_result(name, wl, dev, pattn, st, Ks, args.warmup, peaks, num_sms, l2, barrier,
                                            args.seed + 17)
                except Exception as ex:  # reported, never fatal
                    subs[name] = {"error": str(ex)[:200]}
        try:
            subs["c5_strong_scaling"] = strong_scaling_c5(args, dev, pattn, world, rank, barrier, l2)
        except Exception as ex:
            subs["c5_strong_scaling"] = {"error": str(ex)[:300]}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline(w, args.seed + rank, dev)
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
        "dtype": w.dtype,
        "data": "synthetic",
        "config": {
            "workload": args.workload,
            "seqs": f"{sum(1 for _, q in w.seqs if q > 1)} prefill x {max(qq for _, qq in w.seqs)} tok + "
                    f"{sum(1 for _, q in w.seqs if q == 1)} decode @ ctx {max((c for c, q in w.seqs if q == 1), default=0)}",
            "heads": f"{w.num_q_heads}q/{w.num_kv_heads}kv x d{w.head_dim}",
            "block_size": w.block_size,
            "tokens_per_step_per_gpu": w.num_tokens,
            "parallelism": parallelism_text(args, world, w_global, w),
            **({"comm_backend_test_only": backend} if backend != "nccl" else {}),
            "l2": "inputs > L2 (KV cache %.2f GB/GPU), no flush" % kv_gb,
            "streams": args.streams,
            "flags": args.flags,
            "peaks": peaks["src"] + " (MEASURED_PEAKS.json: HBM %.1f GB/s copy, bf16 %.1f TFLOP/s burst)"
                     % (peaks["hbm"], peaks["bf16"]),
        },
        "roofline": ({k: dominant[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}
                     if dominant else None),
        "roofline_kernels": rl,
        "kernel_ms": kern_ms,
        "instrumented_ms_per_step": ms_instr,
        "clocks": sampler.summary(),
        "e2e": e2e,
        "cuda_graph": graph,
        "gpu_launches": launches_per_step * K,
        "cpu_baseline": cpu,
        "sub_results": subs,
        "gpu_launches_note": "gpu_launches counts the K timed calls of the step-time region",
        "algorithmic": {"prefill_tflop_per_step": work["prefill_flops"] / 1e12,
                        "decode_gb_per_step": work["decode_bytes"] / 1e9,
                        "step_tflops": work["total_flops"] / (ms * 1e-3) / 1e12,
                        "step_gbs": work["total_bytes"] / (ms * 1e-3) / 1e9},
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


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
