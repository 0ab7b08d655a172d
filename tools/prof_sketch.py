"""Run one srt3d_sketch_ex path on a BASELINE config frame (tools only; the target of ncu
captures of the sketch kernels): a warm-up launch, then `--reps` launches.

  python tools/prof_sketch.py [--config C5] [--path 4] [--lanes 0] [--reps 2]"""
import argparse
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
    ap.add_argument("--path", type=int, default=p.PATH_AUTO)
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    f = inputs.make_frame(args.config, n_per_pixel=args.n)
    bins, offs = torch.from_numpy(f.bins).cuda(), torch.from_numpy(f.offsets).cuda()
    z = torch.empty((f.npix, f.m), dtype=torch.complex64, device="cuda")
    for _ in range(1 + args.reps):
        p.srt3d_sketch_ex(bins, offs, f.T, f.m, z=z, total_photons=f.n_photons, path=args.path,
                          lanes_per_pixel=args.lanes)
    torch.cuda.synchronize()
    print("ok", args)


if __name__ == "__main__":
    main()
