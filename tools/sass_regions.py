"""Group an ncu SASS source page (--page source --csv --print-source=sass) into
straight-line regions of equal execution count and report each region's share of
the executed warp instructions and of the stall samples (tools only).

  python tools/sass_regions.py page.csv [top] [out.json]"""
import csv
import json
import sys


def regions(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows[:5]) if r and r[0].startswith("Address")][0]
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    seen = {}
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        a = int(r[0], 16)
        if a not in seen:  # the page may list a kernel's code more than once
            seen[a] = (float(r[ix["Instructions Executed"]] or 0), r[ix["Source"]].strip(),
                       float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    addrs = sorted(seen)
    tot = sum(seen[a][0] for a in addrs) or 1.0
    tsm = sum(seen[a][2] for a in addrs) or 1.0
    out, cur = [], None
    for a in addrs:
        ie, src, smp = seen[a]
        if cur and abs(ie - cur["exec_per_inst"]) <= 0.02 * max(ie, 1.0):
            cur["n_inst"] += 1
            cur["warp_inst"] += ie
            cur["samples"] += smp
            cur["end"] = hex(a)
        else:
            cur = {"start": hex(a), "end": hex(a), "first": src[:60], "exec_per_inst": ie, "n_inst": 1,
                   "warp_inst": ie, "samples": smp}
            out.append(cur)
    for g in out:
        g["inst_share"] = round(g["warp_inst"] / tot, 4)
        g["sample_share"] = round(g["samples"] / tsm, 4)
    return {"total_warp_inst": tot, "total_samples": tsm,
            "regions": sorted(out, key=lambda g: -g["warp_inst"])}


if __name__ == "__main__":
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    r = regions(sys.argv[1])
    r["regions"] = r["regions"][:top]
    s = json.dumps(r, indent=1)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(s)
    print(s)
