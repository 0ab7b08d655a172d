"""Probe of the e2e host path at C5 (tools only): raw pinned H2D rates and
FramePipeline.run_host timings for several chunkings.

  python tools/e2e_probe.py [--config C5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import srt3d_inputs as inputs  # noqa: E402
from paper_2203_00952_b200.pipeline import FramePipeline  # noqa: E402


def ev_time(fn, reps=3, stream=None):
    s = stream or torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--chunks", default="1,2,4,6,8,12,16")
    args = ap.parse_args()
    f = inputs.make_frame(args.config)
    out = {"config": args.config, "n_photons": f.n_photons}
    bins_p = torch.from_numpy(f.bins).pin_memory()
    offs_p = torch.from_numpy(f.offsets).pin_memory()
    t0, a0 = f.theta0()
    t0_p, a0_p = torch.from_numpy(t0).pin_memory(), torch.from_numpy(a0).pin_memory()
    dbin = torch.empty(f.n_photons, dtype=torch.uint16, device="cuda")
    nbytes = 2 * f.n_photons
    ms = ev_time(lambda: dbin.copy_(bins_p, non_blocking=True))
    out["h2d_single_ms"] = ms
    out["h2d_single_gbs"] = nbytes / ms / 1e6
    for nc in (8, 32):
        b = [(f.n_photons * c) // nc for c in range(nc + 1)]

        def chunked():
            for c in range(nc):
                dbin[b[c]:b[c + 1]].copy_(bins_p[b[c]:b[c + 1]], non_blocking=True)

        ms = ev_time(chunked)
        out[f"h2d_{nc}chunks_gbs"] = nbytes / ms / 1e6
    pipe = FramePipeline(f.n_photons, f.npix, f.K, f.T, f.m, f.sigma, f.iters)
    pipe.load_device(torch.from_numpy(f.bins).cuda(), torch.from_numpy(f.offsets).cuda(), torch.from_numpy(t0).cuda(),
                     torch.from_numpy(a0).cuda())
    pipe.capture()
    out["device_step_ms"] = ev_time(pipe.run_device, reps=5, stream=pipe.stream)
    t_out, a_out = torch.empty_like(t0_p).pin_memory(), torch.empty_like(a0_p).pin_memory()
    out["h2d_bytes"] = pipe.h2d_bytes()
    for nc in [int(x) for x in args.chunks.split(",")]:
        def run():
            pipe.run_host(bins_p, offs_p, t0_p, a0_p, t_out, a_out, chunks=nc)
        run()
        torch.cuda.synchronize()
        for steps in (1, 3):
            out[f"run_host_c{nc}_s{steps}_ms"] = ev_time(run, reps=steps, stream=pipe.stream)
        if nc > 1:
            st = {"k": 0}

            def run_chain():
                pipe.run_host(bins_p, offs_p, t0_p, a0_p, t_out, a_out, chunks=nc, chain=st["k"] > 0)
                st["k"] += 1
            for steps in (3, 10):
                st["k"] = 0
                out[f"run_host_c{nc}_chain{steps}_ms"] = ev_time(run_chain, reps=steps, stream=pipe.stream)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
