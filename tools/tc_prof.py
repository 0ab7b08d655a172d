"""Per-role cycle counters of the tensor-core sketch (tools only; needs the TC_PROF build:
SRT3D_VARIANT=prof SRT3D_EXTRA=-DTC_PROF python -m paper_2203_00952_b200.build).

  python tools/tc_prof.py [--config C5] [--lib tools/libsrt3d_prof.so]"""
import argparse
import ctypes
import json
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
    ap.add_argument("--lib", default=os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsrt3d_prof.so"))
    a = ap.parse_args()
    p._lib = p.load_library(a.lib)
    f = inputs.make_frame(a.config, n_per_pixel=a.n)
    bins, offs = torch.from_numpy(f.bins).cuda(), torch.from_numpy(f.offsets).cuda()
    z = torch.empty((f.npix, f.m), dtype=torch.complex64, device="cuda")
    buf = (ctypes.c_ulonglong * 16)()
    run = lambda: p.srt3d_sketch_ex(bins, offs, f.T, f.m, z=z, total_photons=f.n_photons, path=p.PATH_TENSOR)  # noqa
    run()
    torch.cuda.synchronize()
    p._lib.srt3d_debug_tc_prof(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    p._lib.srt3d_debug_tc_prof(buf, 1)
    v = list(buf)
    units = max(v[3], 1)
    names = ["bld_wait_empty", "bld_zero", "bld_scatter", "units", "mma_wait_full", "mma_wait_accempty",
             "epi_wait_accfull", "epi_work"]
    out = {"ms": e0.elapsed_time(e1), "per_unit_cycles": {n: v[i] / units for i, n in enumerate(names) if i != 3},
           "units": units}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
