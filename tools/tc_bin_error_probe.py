"""Per-bin error map of the tensor-core sketch (tools only): one photon per pixel, pixel x holds bin
x, so z[x][j] = exp(i w_j x) exactly; prints the worst entries against the fp64 value and where
they fall in the kernel's row / column split of x.

  python tools/tc_bin_error_probe.py [T ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00952_b200 as p  # noqa: E402


def main():
    for T in [int(a) for a in sys.argv[1:]] or [4613, 8192, 4096, 1000]:
        m = 32
        bins = np.arange(T, dtype=np.uint16)
        offs = np.arange(T + 1, dtype=np.uint32)
        z = p.srt3d_sketch_ex(torch.from_numpy(bins).cuda(), torch.from_numpy(offs).cuda(), T, m,
                              total_photons=T, path=p.PATH_TENSOR).cpu().numpy()
        x = np.arange(T)[:, None].astype(np.float64)
        j = np.arange(1, m + 1)[None, :]
        ref = np.exp(2j * np.pi * ((j * x) % T) / T)
        d = np.abs(z - ref)
        q = max(4, int(np.ceil(np.log2(max(T, 1) / 32))))
        Kb = 1 << q
        print(f"T={T} Kb={Kb} max={d.max():.3e} mean={d.mean():.3e} n>2e-6: {(d > 2e-6).sum()}")
        worst = np.argsort(d.ravel())[::-1][:12]
        for w in worst:
            xi, ji = divmod(int(w), m)
            ahi, khi, alo, klo = xi >> (q + 3), (xi >> 6) & ((1 << (q - 3)) - 1), (xi >> 3) & 7, xi & 7
            print(f"  x={xi} j={ji + 1} d={d[xi, ji]:.3e} a_hi={ahi} k_hi={khi} a_lo={alo} k_lo={klo} "
                  f"Xrow={8 * Kb * ahi + 8 * alo} Xcol={64 * khi + klo} z={z[xi, ji]:.6f} ref={ref[xi, ji]:.6f}")


if __name__ == "__main__":
    main()
