"""Time srt3d_sketch_ex per path / lanes regime on a BASELINE config frame
(tools only), and report the max |delta| between paths.

  python tools/sketch_path_probe.py [--config C5] [--n N] [--reps 5]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00952_b200 as p  # noqa: E402
import srt3d_inputs as inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--only", default=None, help="comma-separated variant names (auto always runs)")
    ap.add_argument("--lib", default=None, help="alternative libsrt3d build (tuning variants)")
    args = ap.parse_args()
    if args.lib:
        p._lib = p.load_library(args.lib)
    f = inputs.make_frame(args.config, n_per_pixel=args.n)
    m = args.m or f.m
    bins, offs = torch.from_numpy(f.bins).cuda(), torch.from_numpy(f.offsets).cuda()
    out = {"config": args.config, "n": args.n, "m": m, "T": f.T, "photons": f.n_photons}
    variants = [("auto", p.PATH_AUTO, 0), ("sorted", p.PATH_PAIRED, 0), ("g4", p.PATH_DIRECT, 4),
                ("g8", p.PATH_DIRECT, 8), ("routed", p.PATH_ROUTED, 0), ("tensor", p.PATH_TENSOR, 0)]
    if args.only:
        variants = [v for v in variants if v[0] in args.only.split(",") or v[0] == "auto"]
    zs = {}
    for name, path, lanes in variants:
        z = torch.empty((f.npix, m), dtype=torch.complex64, device="cuda")
        run = lambda: p.srt3d_sketch_ex(bins, offs, f.T, m, z=z, total_photons=f.n_photons, path=path,  # noqa: E731
                                         lanes_per_pixel=lanes)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        out[name + "_ms"] = ms
        zs[name] = z
    for name in zs:
        out["maxdiff_" + name] = float((zs[name] - zs["auto"]).abs().max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
