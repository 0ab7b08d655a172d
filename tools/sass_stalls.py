"""Stall reasons per SASS instruction from an ncu source page (tools only):
top instructions by long-scoreboard / all samples with their reason breakdown.

  python tools/sass_stalls.py s.csv [reason] [top]"""
import csv
import sys


def main(path, reason="stall_long_sb", top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1] if not rows[0][0].startswith("Address") else rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    recs = []
    for r in rows:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        v = {h: float(r[ix[h]] or 0) for h in reasons}
        recs.append((r[ix["Address"]], r[ix["Source"]], float(r[ix["Instructions Executed"]] or 0), v))
    tot = {h: sum(x[3][h] for x in recs) for h in reasons}
    allt = sum(tot.values())
    print("totals:", {k[6:]: round(100 * v / allt, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v})
    recs.sort(key=lambda x: -x[3][reason])
    for a, s, ie, v in recs[:top]:
        br = {k[6:]: int(x) for k, x in sorted(v.items(), key=lambda kv: -kv[1])[:3] if x}
        print(f"{a[-5:]} ie={ie:.3g} {s[:60]:60s} {br}")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] or []), *([int(sys.argv[3])] if len(sys.argv) > 3 else []))
