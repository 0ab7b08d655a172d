"""Time the NEXT-3 kernels on a BASELINE config's sketch (tools only).
SRT3D_INIT_CUDA_CORES=1 in the environment forces the CUDA-core backprojection.

  python tools/init_probe.py [--config C5] [--N 512] [--K 3] [--min-sep 50]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00952_b200 as p  # noqa: E402
import srt3d_inputs as inputs  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--N", type=int, default=0)
    ap.add_argument("--K", type=int, default=0)
    ap.add_argument("--min-sep", type=int, default=50)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--lib", default=None, help="alternative libsrt3d build (A/B)")
    args = ap.parse_args()
    if args.lib:
        p._lib = p.load_library(args.lib)
    f = inputs.make_frame(args.config)
    N = args.N or 16 * f.m
    K = args.K or f.K
    bins, offs = torch.from_numpy(f.bins).cuda(), torch.from_numpy(f.offsets).cuda()
    z = p.srt3d_sketch(bins, offs, f.T, f.m, total_photons=f.n_photons)
    g = torch.empty((f.npix, N), dtype=torch.float32, device="cuda")
    out = {"config": args.config, "N": N, "K": K, "npix": f.npix, "m": f.m,
           "cuda_cores_forced": os.environ.get("SRT3D_INIT_CUDA_CORES", "0") == "1"}
    out["backproject_ms"] = timed(lambda: p.srt3d_backproject(z, f.sigma, f.T, N, g=g), args.reps)
    out["init_depths_ms"] = timed(lambda: p.srt3d_init_depths(z, f.sigma, f.T, N, K, args.min_sep), args.reps)
    out["init_k1_ms"] = timed(lambda: p.srt3d_init_k1(z, f.sigma, f.T), max(args.reps, 20))
    t, ga, a, c = p.srt3d_init_depths(z, f.sigma, f.T, N, K, args.min_sep)
    torch.cuda.synchronize()
    out["mean_count"] = float(c.float().mean())
    out["checksum_t"] = float(t.double().sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
