"""Time the fused gradient step (srt3d_sketch_grad_step, the kernel the bench's
iteration loop runs) on a C5-shaped frame (tools only): in a 200-iteration
CUDA graph (L2-warm theta) and as single launches after an L2 flush (cold),
median / min over reps.  z is the expected sketch of a random theta* plus
noise (the kernel's cost does not depend on the values).

  python tools/grad_probe.py [--npix 262144] [--m 32] [--K 3] [--lib other.so]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_00952_b200 as p  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--npix", type=int, default=512 * 512)
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--K", type=int, default=3)
    ap.add_argument("--T", type=int, default=8192)
    ap.add_argument("--sigma", type=float, default=6.0)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--lib", default=None)
    a = ap.parse_args()
    if a.lib:
        p._lib = p.load_library(a.lib)
    g = torch.Generator(device="cuda").manual_seed(5)
    t = torch.rand((a.npix, a.K), device="cuda", generator=g) * a.T
    al = torch.rand((a.npix, a.K), device="cuda", generator=g) * 0.9 + 0.05
    z = p.srt3d_expected_sketch(t, al, a.sigma, a.T, a.m)
    z += 0.01 * torch.randn(z.shape, dtype=torch.complex64, device="cuda", generator=g)
    t0, a0 = t + 10.0, al.clone()
    tt, aa = t0.clone(), a0.clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            p.srt3d_sketch_grad_step(z, tt, aa, a.sigma, a.T, a.m, stream=s)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        tt.copy_(t0)
        aa.copy_(a0)
        for _ in range(a.iters):
            p.srt3d_sketch_grad_step(z, tt, aa, a.sigma, a.T, a.m, stream=s)
    loop = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            graph.replay()
            e1.record(s)
        s.synchronize()
        loop.append(e0.elapsed_time(e1) * 1000.0 / a.iters)
    # the loop alternating two copies of z (134 MB > L2): z cannot stay L2-resident
    z2 = z.clone()
    g_alt = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_alt, stream=s):
        tt.copy_(t0)
        aa.copy_(a0)
        for it in range(a.iters):
            p.srt3d_sketch_grad_step(z if it % 2 == 0 else z2, tt, aa, a.sigma, a.T, a.m, stream=s)
    alt = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g_alt.replay()
            e1.record(s)
        s.synchronize()
        alt.append(e0.elapsed_time(e1) * 1000.0 / a.iters)
    del g_alt
    flush = torch.ones(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sink = torch.empty(1, dtype=torch.float32, device="cuda")
    cold, dirty = [], []
    for _ in range(a.reps):  # dirty-L2 cold: the flush WRITES 512 MB (L2 full of dirty lines)
        with torch.cuda.stream(s):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            p.srt3d_sketch_grad_step(z, tt, aa, a.sigma, a.T, a.m, stream=s)
            e1.record(s)
        s.synchronize()
        dirty.append(e0.elapsed_time(e1) * 1000.0)
    for _ in range(a.reps):  # clean-L2 cold: the flush READS 512 MB (L2 full of clean lines)
        with torch.cuda.stream(s):
            sink.copy_(flush.sum().reshape(1))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            p.srt3d_sketch_grad_step(z, tt, aa, a.sigma, a.T, a.m, stream=s)
            e1.record(s)
        s.synchronize()
        cold.append(e0.elapsed_time(e1) * 1000.0)
    empty, warm1 = [], []
    for _ in range(a.reps):  # the same clean flush, then a 1-element kernel: event + launch overhead
        with torch.cuda.stream(s):
            sink.copy_(flush.sum().reshape(1))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            sink.add_(1.0)
            e1.record(s)
        s.synchronize()
        empty.append(e0.elapsed_time(e1) * 1000.0)
    for _ in range(a.reps):  # a single launch right after another one (L2-warm, not in a graph)
        with torch.cuda.stream(s):
            p.srt3d_sketch_grad_step(z, tt, aa, a.sigma, a.T, a.m, stream=s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            p.srt3d_sketch_grad_step(z, tt, aa, a.sigma, a.T, a.m, stream=s)
            e1.record(s)
        s.synchronize()
        warm1.append(e0.elapsed_time(e1) * 1000.0)
    # cold per launch inside CUDA graphs (launch overhead hidden): [flush, step] x N minus [flush] x N
    # one float per 2 MB page of z and theta (warms the TLBs, leaves L2 ~empty of them)
    zf = torch.view_as_real(z).reshape(-1)
    pages = [x[:: (2 << 20) // 4] for x in (zf, tt.reshape(-1), aa.reshape(-1))]
    psink = torch.zeros(1, device="cuda")

    def graph_ms(with_step, n=20, touch=False, icache=False):
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=s):
            for _ in range(n):
                sink.copy_(flush.sum().reshape(1))
                if touch:
                    for pg in pages:
                        psink.add_(pg.sum())
                if icache:  # one 64-pixel launch of the same kernel: its code into the caches
                    p.srt3d_sketch_grad_step(z[:64], tt[:64], aa[:64], a.sigma, a.T, a.m, stream=s)
                for _ in range(with_step):
                    p.srt3d_sketch_grad_step(z, tt, aa, a.sigma, a.T, a.m, stream=s)
        res = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                g2.replay()
                e1.record(s)
            s.synchronize()
            res.append(e0.elapsed_time(e1))
        del g2
        return sorted(res)[2], n
    gw, n_g = graph_ms(1)
    gf, _ = graph_ms(0)
    g2w, _ = graph_ms(2)
    graph_cold = (gw - gf) * 1000.0 / n_g
    graph_second = (g2w - gw) * 1000.0 / n_g  # the launch right after a cold one (theta L2-warm)
    gtw, _ = graph_ms(1, touch=True)
    gtf, _ = graph_ms(0, touch=True)
    graph_cold_tlb = (gtw - gtf) * 1000.0 / n_g  # cold L2, TLB entries of z / theta warmed
    pages[:] = [tt.reshape(-1), aa.reshape(-1)]  # now: read all of theta (6 MB) into L2 after the flush
    gqw, _ = graph_ms(1, touch=True)
    gqf, _ = graph_ms(0, touch=True)
    graph_cold_theta_warm = (gqw - gqf) * 1000.0 / n_g
    giw, _ = graph_ms(1, icache=True)
    gif, _ = graph_ms(0, icache=True)
    graph_cold_icache_warm = (giw - gif) * 1000.0 / n_g

    empty.sort()
    warm1.sort()
    loop.sort()
    cold.sort()
    dirty.sort()
    nbytes = a.npix * (8 * a.m + 16 * a.K)
    print(json.dumps({"npix": a.npix, "m": a.m, "K": a.K, "lib": a.lib, "loop_us_median": loop[len(loop) // 2],
                      "loop_us_min": loop[0], "cold_us_median": cold[len(cold) // 2], "cold_us_min": cold[0],
                      "dirty_cold_us_median": dirty[len(dirty) // 2], "dirty_cold_us_min": dirty[0],
                      "empty_after_flush_us_median": empty[len(empty) // 2],
                      "warm_single_us_median": warm1[len(warm1) // 2],
                      "cold_in_graph_us": graph_cold, "second_after_cold_in_graph_us": graph_second,
                      "cold_tlb_warm_in_graph_us": graph_cold_tlb, "cold_theta_warm_in_graph_us": graph_cold_theta_warm,
                      "cold_code_warm_in_graph_us": graph_cold_icache_warm,
                      "loop_two_z_us_median": sorted(alt)[2],
                      "cold_frac_hbm": nbytes / (cold[len(cold) // 2] * 1e-6) / 6545.3e9,
                      "loop_frac_hbm": nbytes / (loop[len(loop) // 2] * 1e-6) / 6545.3e9}))


if __name__ == "__main__":
    main()
