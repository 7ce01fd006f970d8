"""Summarise gpurun_out/ ncu artefacts into profiles/<round>/ (text + traffic.json).

  python scripts/profile_summary.py r01
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import load  # noqa: E402

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "SM_A.TriageCompute.sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals) if h in METRICS}


def main(rnd):
    src = os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    traffic = {}
    lines = []
    for f in sorted(os.listdir(src)):
        if f.startswith("ncu_") and f.endswith(".csv") and f != "ncu_k1_tensor.csv":
            wl = f[4:-4]
            shutil.copy(os.path.join(src, f), os.path.join(dst, f"launches_{wl}.csv"))
            agg = load(os.path.join(src, f))
            tot = sum(sum(v.get("gpu__time_duration.sum", [0])) for v in agg.values())
            lines.append(f"## launch list {wl} (ncu --metrics gpu__time_duration.sum,dram__bytes_*; cold-cache, serialised)")
            for k, v in agg.items():
                t = v.get("gpu__time_duration.sum", [0])
                rd = v.get("dram__bytes_read.sum", [0])
                wr = v.get("dram__bytes_write.sum", [0])
                n = len(t)
                lines.append(f"  {k:12s} launches {n:3d} mean {sum(t)/n/1e3:9.2f} us share {sum(t)/tot:6.1%} "
                             f"dram rd {sum(rd)/n/1e6:9.2f} MB wr {sum(wr)/n/1e6:8.2f} MB")
                name = {"k1_prefill": "prefill", "k2_decode": "decode", "k2w_decode": "decode", "k3_reduce": "reduce",
                        "k4_generic": "generic", "k5_metadata": "metadata"}.get(k, k)
                traffic.setdefault(wl, {})[name] = (sum(rd) + sum(wr)) / n
    for rep in ("k1_c3_full", "k1_c3p_full", "k2_c2_full", "k2_c4_full", "k2_sm36", "k2w_c2_full", "k2w_c4_full",
                "k2w_sm36_main", "k3_c4_full", "k6_c3_full"):
        path = os.path.join(src, rep + ".ncu-rep")
        if os.path.exists(path):
            shutil.copy(path, os.path.join(dst, rep + ".ncu-rep"))
            lines.append(f"## ncu --set full {rep}")
            for k, (v, u) in raw_metrics(path).items():
                lines.append(f"  {k} = {v} {u}")
    for f in sorted(os.listdir(src)):
        if f.startswith("bench_") and f.endswith(".json"):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    open(os.path.join(dst, "summary.txt"), "w").write("\n".join(lines) + "\n")
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old.update(traffic)
    json.dump(old, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
