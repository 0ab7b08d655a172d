"""Launch srt3d_bucket_events once on a C5-sized random event stream (tools only; for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_00952_b200 as p  # noqa: E402

npix = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
N = npix * (int(sys.argv[2]) if len(sys.argv) > 2 else 1000)
pix = torch.randint(0, npix, (N,), device="cuda", dtype=torch.int32).view(torch.uint32)
b = torch.randint(0, 8192, (N,), device="cuda", dtype=torch.int16).view(torch.uint16)
p.srt3d_bucket_events(pix, b, npix)
torch.cuda.synchronize()
print("ok")
