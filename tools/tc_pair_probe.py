"""Tensor-core sketch of one pixel holding a given list of bins, printed against the fp64 sketch
per frequency (tools only):  python tools/tc_pair_probe.py T m bin [bin ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00952_b200 as p  # noqa: E402

T, m = int(sys.argv[1]), int(sys.argv[2])
for spec in sys.argv[3:]:
    b = np.array([int(x) for x in spec.split(",")], dtype=np.uint16)
    o = np.array([0, len(b)], dtype=np.uint32)
    z = p.srt3d_sketch_ex(torch.from_numpy(b).cuda(), torch.from_numpy(o).cuda(), T, m, total_photons=len(b),
                          path=p.PATH_TENSOR).cpu().numpy()[0]
    j = np.arange(1, m + 1)
    ref = np.exp(2j * np.pi * ((j[:, None] * b[None, :].astype(np.int64)) % T) / T).mean(1)
    d = z - ref
    print(spec, "max", f"{np.abs(d).max():.3e}", " ".join(f"{j_}:{d_.real:+.1e}{d_.imag:+.1e}i" for j_, d_ in zip(j, d)))
