"""Summarise an ncu source page (--page source --csv --print-source=sass) by SASS region
(tools only): instructions executed, average active threads and stall samples per block
of consecutive addresses, plus the top-N instructions by stall samples.

  ncu -i rep --page source --csv --print-source=sass > s.csv; python tools/ncu_sass_hot.py s.csv"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[0].startswith("0x") and not r[0].isdigit():
            continue
        try:
            addr = int(r[ix["Address"]], 16) if r[ix["Address"]].startswith("0x") else int(r[ix["Address"]])
        except ValueError:
            continue
        ie = float(r[ix["Instructions Executed"]] or 0)
        te = float(r[ix["Thread Instructions Executed"]] or 0)
        st = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        recs.append((addr, r[ix["Source"]], ie, te, st))
    tot_ie = sum(x[2] for x in recs)
    tot_st = sum(x[4] for x in recs)
    print(f"total warp instructions {tot_ie:.4g}, stall samples {tot_st:.4g}")
    # regions of 64 instructions
    blk = {}
    for a, s, ie, te, st in recs:
        b = a // 0x400
        d = blk.setdefault(b, [0, 0, 0, s])
        d[0] += ie
        d[1] += te
        d[2] += st
    print("region      warp-inst%   thr/inst  stall%   first")
    for b in sorted(blk):
        ie, te, st, s = blk[b]
        if ie / tot_ie > 0.005 or st / max(tot_st, 1) > 0.005:
            print(f"{b * 0x400:#07x}  {100 * ie / tot_ie:8.2f}  {te / max(ie, 1):8.1f}  {100 * st / max(tot_st, 1):6.2f}   {s[:60]}")
    print("top instructions by stall samples:")
    for a, s, ie, te, st in sorted(recs, key=lambda x: -x[4])[:top]:
        print(f"{a:#07x} {100 * st / max(tot_st, 1):5.2f}% ie={ie:.3g} thr={te / max(ie, 1):4.1f}  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
