"""Launch srt3d_bucket_events on a C5-sized random event stream (tools only; for ncu),
then time it with CUDA events (--time).

  python tools/bucket_probe.py [npix] [events_per_pixel] [--time]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_00952_b200 as p  # noqa: E402

if "--lib" in sys.argv:  # alternative build (A/B)
    _i = sys.argv.index("--lib")
    p._lib = p.load_library(sys.argv[_i + 1])
    del sys.argv[_i:_i + 2]
args = [a for a in sys.argv[1:] if not a.startswith("--")]
npix = int(args[0]) if len(args) > 0 else 262144
N = npix * (int(args[1]) if len(args) > 1 else 1000)
pix = torch.randint(0, npix, (N,), device="cuda", dtype=torch.int32).view(torch.uint32)
b = torch.randint(0, 8192, (N,), device="cuda", dtype=torch.int16).view(torch.uint16)
offs, out, _ = p.srt3d_bucket_events(pix, b, npix)
torch.cuda.synchronize()
if "--time" in sys.argv:
    scratch = torch.empty(p.srt3d_bucket_scratch_words(npix, N), dtype=torch.uint32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        p.srt3d_bucket_events(pix, b, npix, offsets=offs, out=out, scratch=scratch)
    e0.record()
    reps = 10
    for _ in range(reps):
        p.srt3d_bucket_events(pix, b, npix, offsets=offs, out=out, scratch=scratch)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"npix={npix} events={N} ms={ms:.4f} events/s={N / ms * 1e3:.3e}")
else:
    print("ok")
