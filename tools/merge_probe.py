"""Time srt3d_sketch_merge on a C5-shaped sketch (tools only):  python tools/merge_probe.py [--lib x.so]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00952_b200 as p  # noqa: E402

if "--lib" in sys.argv:
    p._lib = p.load_library(sys.argv[sys.argv.index("--lib") + 1])
npix, m = 512 * 512, 32
g = torch.Generator(device="cuda").manual_seed(1)
za = torch.randn((npix, m), dtype=torch.complex64, device="cuda", generator=g)
zb = torch.randn((npix, m), dtype=torch.complex64, device="cuda", generator=g)
na = torch.randint(0, 2000, (npix,), device="cuda", dtype=torch.int32, generator=g).view(torch.uint32)
nb = torch.randint(0, 2000, (npix,), device="cuda", dtype=torch.int32, generator=g).view(torch.uint32)
zo, no = torch.empty_like(za), torch.empty_like(na)
for _ in range(3):
    p.srt3d_sketch_merge(za, na, zb, nb, z_out=zo, n_out=no)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    p.srt3d_sketch_merge(za, na, zb, nb, z_out=zo, n_out=no)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
b = 3 * npix * (8 * m + 4)
print(json.dumps({"merge_ms": ms, "gbs": b / ms / 1e6, "frac_hbm": b / ms / 1e6 / 6545.3}))
