"""Launch each hot kernel a few times on a BASELINE config (no graphs) so ncu
can capture them:  python tools/prof_kernels.py C5 [--iters 3] [--n 1000000]
Exits 0 on success (required before running it under ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2203_00952_b200 as p  # noqa: E402
import srt3d_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="C5", nargs="?")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--n", type=int, default=1000000)
    ap.add_argument("--skip-sketch", action="store_true")
    ap.add_argument("--unfused", action="store_true")
    ap.add_argument("--next", action="store_true", help="also launch the NEXT-2/3/4 kernels once")
    a = ap.parse_args()
    f = srt3d_inputs.make_frame(a.config, n_per_pixel=a.n if a.config == "C4" else None)
    bins = torch.from_numpy(f.bins).cuda()
    offs = torch.from_numpy(f.offsets).cuda()
    t0, a0 = (torch.from_numpy(x).cuda() for x in f.theta0())
    z = p.srt3d_sketch(bins, offs, f.T, f.m, total_photons=f.n_photons)
    if not a.skip_sketch:
        for _ in range(2):
            p.srt3d_sketch(bins, offs, f.T, f.m, z=z, total_photons=f.n_photons)
    if f.iters:
        t, al = t0.clone(), a0.clone()
        for _ in range(a.iters):
            if a.unfused:
                gt, ga, _ = p.srt3d_sketch_grad(z, t, al, f.sigma, f.T, f.m)
                p.srt3d_descent_update(t, al, gt, ga, f.sigma, f.T, f.m)
            else:
                p.srt3d_sketch_grad_step(z, t, al, f.sigma, f.T, f.m)
    if a.next and f.iters:
        t, al = t0.clone(), a0.clone()
        p.srt3d_fit_pixelwise(z, t, al, f.sigma, f.T, f.m, f.iters)
        p.srt3d_init_depths(z, f.sigma, f.T, min(4096, 16 * f.m), f.K, 50)
        p.srt3d_init_k1(z, f.sigma, f.T)
        n = (offs[1:].to(torch.int64) - offs[:-1].to(torch.int64)).to(torch.int32).view(torch.uint32).contiguous()
        p.srt3d_sketch_merge(z, n, z.clone(), n.clone())
    torch.cuda.synchronize()
    print("ok", f.name, f.n_photons)


if __name__ == "__main__":
    main()
