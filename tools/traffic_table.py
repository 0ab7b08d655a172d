"""Build profiles/traffic.json (DRAM read+write bytes per launch, per config and entry point)
from the round's ncu summaries (tools only):  python tools/traffic_table.py r02"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ENTRY = [("sketch_tc", "srt3d_sketch"), ("sketch_routed", "srt3d_sketch"), ("sketch_hist", "srt3d_sketch"), ("sketch_kernel", "srt3d_sketch"),
         ("grad_kernel", "srt3d_sketch_grad_step"), ("fit_kernel", "srt3d_fit_pixelwise"),
         ("bp_tc_kernel", "srt3d_init_depths"), ("init_k1", "srt3d_init_k1"), ("merge_kernel", "srt3d_sketch_merge")]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    out = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (median over the captured launches) "
                    "from one `ncu --set full` capture per config (ncu flushes caches between replays: L2-cold). "
                    f"Sources: profiles/{tag}_ncu_*.json (tools/profile_round2.sh); C5 bucket_events = the sum of "
                    "its three passes."}
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"{tag}_ncu_*.json"))):
        name = os.path.basename(f)[len(tag) + 5:-5]
        launches = json.load(open(f))
        launches = launches if isinstance(launches, list) else launches.get("launches", [launches])
        if name == "bucket":
            out.setdefault("C5", {})["srt3d_bucket_events"] = sum(x["dram_bytes_per_launch"] for x in launches)
            continue
        cfg = name if not name.startswith("C4_") else "C4@1e%d" % (len(name) - 4)
        per = {}
        for x in launches:
            for key, entry in ENTRY:
                if key in x["kernel"]:
                    per.setdefault(entry, []).append(x["dram_bytes_per_launch"])
                    break
        d = out.setdefault(cfg, {})
        for entry, v in per.items():
            d[entry] = sorted(v)[len(v) // 2]
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
