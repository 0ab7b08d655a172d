"""A12 margin of the gradient kernels over many random pixels (tools only): worst
|d| / (1e-4 |ref| + 1e-6 S) per component against the fp64 oracle.

  python tools/a12_probe.py T m K npix [seed]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2203_00952_b200 as p  # noqa: E402
from test_gpu_parity import _grad_S  # noqa: E402

T, m, K, npix = (int(x) for x in sys.argv[1:5])
seed = int(sys.argv[5]) if len(sys.argv) > 5 else 0
rng = np.random.default_rng(seed)
sigma = 2.0
z = (rng.normal(size=(npix, m)) + 1j * rng.normal(size=(npix, m))).astype(np.complex64) * 0.3
t = rng.uniform(0, T, (npix, K)).astype(np.float32)
a = rng.uniform(0.05, 1, (npix, K)).astype(np.float32)
dz, dt, da = (torch.from_numpy(x).cuda() for x in (z, t, a))
gt, ga, L = (x.cpu().numpy() for x in p.srt3d_sketch_grad(dz, dt, da, sigma, T, m))
go = oracle.sketch_grad(z, t, a, sigma, T, m)
S_L, S_a, S_t = _grad_S(z, a, sigma, T, m)
out = {}
for name, g, o, S in (("grad_t", gt, go[0], S_t), ("grad_alpha", ga, go[1], np.broadcast_to(S_a[:, None], ga.shape))):
    d = np.abs(g.astype(np.float64) - o)
    lim = 1e-4 * np.abs(o) + 1e-6 * S
    out[name] = float((d / lim).max())
print({"T": T, "m": m, "K": K, "npix": npix, **out})
