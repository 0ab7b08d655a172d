"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch
list: per kernel name, launch count, total / mean device time and share of the
total.  Usage: python tools/launch_summary.py launches.csv [out.json]"""
import csv
import json
import sys
from collections import defaultdict


def summarise(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, im, iv, iu = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0]
        us = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        agg[name][0] += 1
        agg[name][1] += us
    total = sum(v[1] for v in agg.values())
    out = [{"kernel": k, "launches": n, "total_us": round(t, 2), "mean_us": round(t / n, 3),
            "share": round(t / total, 4)} for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    return {"total_us": round(total, 2), "kernels": out}


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    txt = json.dumps(s, indent=1)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(txt + "\n")
    print(txt)
