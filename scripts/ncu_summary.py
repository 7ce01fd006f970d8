"""Summarise an ncu --csv launch list: per kernel name, launches, mean duration, dram bytes per launch."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    agg = defaultdict(lambda: defaultdict(list))
    for i, m in per.items():
        n = names[i]
        short = next((k for k in ("k1_prefill", "k2w_decode", "k2_decode", "k3_reduce", "k4_generic", "k5_metadata") if k in n), n[:40])
        for k, v in m.items():
            agg[short][k].append(v)
    return agg


if __name__ == "__main__":
    for path in sys.argv[1:]:
        agg = load(path)
        tot = sum(sum(v.get("gpu__time_duration.sum", [0])) for v in agg.values())
        print(path)
        for k, v in agg.items():
            t = v.get("gpu__time_duration.sum", [0])
            rd = v.get("dram__bytes_read.sum", [0])
            wr = v.get("dram__bytes_write.sum", [0])
            n = len(t)
            print(f"  {k:12s} launches {n:3d}  mean {sum(t)/n/1e3:9.2f} us  share {sum(t)/tot:6.1%}  "
                  f"dram rd {sum(rd)/n/1e6:9.2f} MB  wr {sum(wr)/n/1e6:8.2f} MB  "
                  f"-> {(sum(rd)+sum(wr))/max(sum(t),1):7.1f} GB/s")
