"""One small call of every libsrt3d.so entry point (tools only; the target for
compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck where the tool
is available — SURVEY §4 T5; it is closed on this round's GPU pool).
Ragged C1-sized inputs with empty pixels, misaligned CSR base, every sketch
path (grouped direct at G = 4..32, paired, bin-count), m > 32 (two passes),
the gradient / fused step / fit / update, NEXT-3 and NEXT-4."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_00952_b200 as p  # noqa: E402
import srt3d_inputs  # noqa: E402


def main():
    dev = "cuda"
    T, m = 1024, 40
    bins, offs = srt3d_inputs.random_csr(npix=97, T=T, max_n=700, seed=3)
    pad = np.concatenate([np.zeros(1, np.uint16), bins])  # 2-byte-misaligned base
    db = torch.from_numpy(pad).to(dev)[1:]
    do = torch.from_numpy(offs).to(dev)
    n = int(offs[-1])
    for g in (4, 8, 16, 32):
        p.srt3d_sketch_ex(db, do, T, m, total_photons=n, path=p.PATH_DIRECT, lanes_per_pixel=g)
    p.srt3d_sketch_ex(db, do, T, m, total_photons=n, path=p.PATH_PAIRED)
    p.srt3d_sketch_ex(db, do, T, m, total_photons=n, path=p.PATH_BINCOUNT)
    z = p.srt3d_sketch(db, do, T, 32, total_photons=n)
    p.srt3d_debug_phase_index(db[:100].contiguous(), T, 8)
    p.srt3d_check_csr(db, do, T)
    t, a = (torch.from_numpy(x).to(dev) for x in srt3d_inputs.random_theta(97, 3, T, seed=1))
    sigma = 2.0
    p.srt3d_expected_sketch(t, a, sigma, T, 32)
    gt, ga, L = p.srt3d_sketch_grad(z, t, a, sigma, T, 32)
    p.srt3d_descent_update(t, a, gt, ga, sigma, T, 32)
    p.srt3d_sketch_grad_step(z, t, a, sigma, T, 32)
    p.srt3d_fit_pixelwise(z, t.clone(), a.clone(), sigma, T, 32, 3)
    z7 = p.srt3d_sketch(db, do, T, 7, total_photons=n)  # odd m: generic layouts
    p.srt3d_sketch_grad_step(z7, t, a, sigma, T, 7)
    p.srt3d_backproject(z, sigma, T, 100)
    p.srt3d_init_depths(z, sigma, T, 64, 3, 20)
    p.srt3d_init_k1(z, sigma, T)
    cnt = torch.from_numpy(np.diff(offs.astype(np.int64)).astype(np.uint32)).to(dev)
    p.srt3d_sketch_merge(z, cnt, z.clone(), cnt.clone())
    ev_p = torch.randint(0, 120, (5000,), device=dev, dtype=torch.int32).view(torch.uint32)
    ev_b = torch.randint(0, T, (5000,), device=dev, dtype=torch.int16).view(torch.uint16)
    p.srt3d_bucket_events(ev_p, ev_b, 100)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
