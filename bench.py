#!/usr/bin/env python
"""bench.py — SRT3D hot path on B200: one step = sketch one synthetic frame
(Eq. 3) + the config's sketched-gradient iterations (Eq. 6/8 data step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5]
                  [--n-per-pixel 1000000 (C4 only)] [--impl srt3d|reference]

Default workload: BASELINE.json configs[4] (C5: 512x512 px, T=8192, K=3,
1000 photons/px at SBR 0.01, m=32, 200 iterations) — the largest config that
exercises both kernels (DESIGN.md §7 explains the choice).  Inputs are
seeded synthetic frames (srt3d_inputs) standing in for the paper's datasets.

Multi-GPU (torchrun): pixels are independent (no data-path collective);
every rank processes its own frame of the same config ("scaling": "weak"),
timed with CUDA events between barriers, max over ranks.

Rank 0 prints ONE JSON line.  --impl reference times the fp64 CPU oracle on
the host cores instead (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP32_LANES_PER_SM = 128  # FP32 FMA lanes per SM (B200)
METRIC = "photons/s sketched (GB/s vs HBM peak); sketched-gradient pixel-iters/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="srt3d", choices=["srt3d", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n-per-pixel", type=int, default=1000000, help="C4 photons per pixel")
    ap.add_argument("--unfused", action="store_true", help="separate grad + update kernels")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample duration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None, help="frames in the e2e timed region (default: --steps)")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="pixel blocks pipelined H2D/compute in the e2e path")
    ap.add_argument("--no-init", action="store_true", help="skip the NEXT-3 initialisation timings")
    ap.add_argument("--init-grid", type=int, default=0, help="backprojection grid points (default 16 m)")
    ap.add_argument("--init-min-sep", type=int, default=50, help="minimum separation of initial depths (bins)")
    ap.add_argument("--no-stream", action="store_true", help="skip the NEXT-4 bucketing / merge timings")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the per-config sketch / gradient sweep (C1-C3, C4@1e2..1e6; SURVEY §8(d))")
    ap.add_argument("--sweep-configs", default="C4@1e6,C1,C2,C3,C4@1e2,C4@1e3,C4@1e4,C4@1e5",
                    help="comma list of sweep workloads (C4@<n> = C4 at n photons/pixel)")
    ap.add_argument("--sketch-reps", type=int, default=20, help="timed sketch reps per workload (5 at C4@1e6)")
    args = ap.parse_args()
    if args.e2e_steps is None:
        args.e2e_steps = args.steps
    return args


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index: int):
        self.dev = dev_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()
        time.sleep(0.25)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ oracle (CPU)
def oracle_step_sample(frame, seconds: float, single_core: bool = False):
    """Time the fp64 oracle (as it stands) on a bounded sample of the frame:
    sketch of npix_s pixels + the config's iterations on those pixels."""
    import oracle

    oracle.build()
    cores = oracle.max_threads()

    def run(npix_s):
        idx = np.arange(npix_s)
        offs = frame.offsets[: npix_s + 1].astype(np.int64)
        bins = frame.bins[offs[0]:offs[-1]]
        offs = (offs - offs[0]).astype(np.uint32)
        t0, a0 = frame.theta0()
        t, a = t0[idx].astype(np.float64), a0[idx].astype(np.float64)
        t_start = time.perf_counter()
        z = oracle.sketch(bins, offs, frame.T, frame.m)
        for _ in range(frame.iters):
            gt, ga, _ = oracle.sketch_grad(z, t, a, frame.sigma, frame.T, frame.m)
            t, a = oracle.descent_update(t, a, gt, ga, frame.sigma, frame.T, frame.m, eta=0.5)
        dt = time.perf_counter() - t_start
        return dt, int(offs[-1])

    n = min(frame.npix, 64)
    dt, ph = run(n)
    while dt < 0.05 * seconds and n < frame.npix:
        n = min(frame.npix, n * 4)
        dt, ph = run(n)
    if dt < seconds and n < frame.npix:
        n = min(frame.npix, max(n, int(n * seconds / max(dt, 1e-6))))
        dt, ph = run(n)
    out = {"seconds": dt, "photons": ph, "pixels": n, "cores": cores, "cpu_model": _cpu_model(),
           "sample": f"first {n} of {frame.npix} pixels ({ph} photons): oracle sketch + {frame.iters} "
                     f"fp64 gradient/update iterations"}
    if single_core and cores > 1:  # also one core, on a proportionally smaller sample
        oracle.set_threads(1)
        try:
            n1 = max(1, n // cores)
            dt1, ph1 = run(n1)
            out["one_core"] = {"value": ph1 / dt1, "unit": "photons/s", "pixels": n1, "seconds": dt1}
        finally:
            oracle.set_threads(cores)
    return out


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def make_frame(args, rank: int):
    import srt3d_inputs

    if args.config == "C4":
        f = srt3d_inputs.make_frame("C4", n_per_pixel=args.n_per_pixel,
                                    seed=None if rank == 0 else 104 + 1000 * rank)
    else:
        seed = None if rank == 0 else srt3d_inputs.CONFIGS[args.config]["seed"] + 1000 * rank
        f = srt3d_inputs.make_frame(args.config, seed=seed)
    return f


def config_obj(f, args):
    return {"workload": f"{f.name}: {f.rows}x{f.cols} px, T={f.T}, K={f.K}, m={f.m}, sigma={f.sigma}, "
                        f"{'fixed ' + str(args.n_per_pixel) if args.config == 'C4' else 'Poisson mean ' + str(f.lam)}"
                        f" photons/px, SBR={f.sbr}, {f.iters} gradient iterations",
            "npix": f.npix, "photons_per_frame": f.n_photons, "T": f.T, "m": f.m, "K": f.K, "sigma": f.sigma,
            "iters": f.iters, "seed": f.seed, "recipe": f.recipe,
            "l2": "photon input per step larger than L2 (not flushed); in the iteration loop theta stays L2-resident "
                  "and z (67 MB) partly (two-z loop: 14.7 vs 13.6 us per iteration); the gradient's headline "
                  "fraction is its L2-flushed launch",
            "parallelism": f"dp{args.gpus} (independent frames per GPU)"}


# ------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    f = make_frame(args, 0)
    per_step = max(1.0, args.cpu_seconds / max(args.steps, 1))
    for _ in range(args.warmup if args.warmup < 1 else 1):
        oracle_step_sample(f, min(per_step, 1.0))
    times, photons, info = [], [], None
    for _ in range(args.steps):
        info = oracle_step_sample(f, per_step)
        times.append(info["seconds"])
        photons.append(info["photons"])
    value = sum(photons) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "photons/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_obj(f, args),
            "cpu_baseline": {"value": value, "unit": "photons/s", "cores": info["cores"], "kind": "oracle",
                             "sample": info["sample"], "cpu_model": info["cpu_model"]},
            "e2e": {"value": value, "unit": "photons/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ timing helpers
def _l2_flush(torch, buf, sink, s):
    """Evict L2 by READING a buffer of twice its size (clean lines: no write-back lands on the
    next kernel)."""
    with torch.cuda.stream(s):
        torch.sum(buf, dim=0, out=sink[0])


def time_sketch(torch, srt3d, bins, offs, z, T, m, hint, reps, s, flush=None):
    """Median / min over reps of one srt3d_sketch launch (CUDA events on s); the L2 is flushed
    before every rep when `flush` = (buffer, sink) is given (inputs smaller than L2)."""
    with torch.cuda.stream(s):
        for _ in range(2):  # warm-up
            srt3d.srt3d_sketch(bins, offs, T, m, z=z, total_photons=hint, stream=s)
    times = []
    for _ in range(reps):
        if flush is not None:
            _l2_flush(torch, flush[0], flush[1], s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            srt3d.srt3d_sketch(bins, offs, T, m, z=z, total_photons=hint, stream=s)
            e1.record(s)
        times.append((e0, e1))
    s.synchronize()
    ms = sorted(e0.elapsed_time(e1) for e0, e1 in times)
    return statistics.median(ms), ms[0]


def time_grad(torch, srt3d, z, t0, a0, sigma, T, m, iters, s, flush, reps=20):
    """The fused gradient step: per-iteration time inside an `iters`-launch CUDA graph
    (L2-warm theta; median of 5 replays) and single launches after an L2 flush (cold; median /
    min of reps)."""
    t, a = t0.clone(), a0.clone()
    with torch.cuda.stream(s):
        for _ in range(3):
            srt3d.srt3d_sketch_grad_step(z, t, a, sigma, T, m, 0.5, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        t.copy_(t0)
        a.copy_(a0)
        for _ in range(iters):
            srt3d.srt3d_sketch_grad_step(z, t, a, sigma, T, m, 0.5, stream=s)
    loop = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        s.synchronize()
        loop.append(e0.elapsed_time(e1) / iters)
    cold = []
    for _ in range(reps):
        _l2_flush(torch, flush[0], flush[1], s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            srt3d.srt3d_sketch_grad_step(z, t, a, sigma, T, m, 0.5, stream=s)
            e1.record(s)
        cold.append((e0, e1))
    s.synchronize()
    cms = sorted(e0.elapsed_time(e1) for e0, e1 in cold)
    del g

    # the same cold launch without its launch latency: CUDA graphs of n x [flush, step] and
    # n x [flush], events around each replay; per-launch cold time = the difference / n
    def graph_ms(with_step, n=20):
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=s):
            for _ in range(n):
                _l2_flush(torch, flush[0], flush[1], s)
                if with_step:
                    srt3d.srt3d_sketch_grad_step(z, t, a, sigma, T, m, 0.5, stream=s)
        res = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                g2.replay()
                e1.record(s)
            s.synchronize()
            res.append(e0.elapsed_time(e1))
        del g2
        return statistics.median(res) / n
    in_graph = graph_ms(True) - graph_ms(False)
    return statistics.median(loop), min(loop), statistics.median(cms), cms[0], in_graph


def sketch_work(srt3d, npix, T, m, n_photons):
    """Algorithmic bytes and flops of one sketch launch: B = 2n + 4(npix+1) + 8 m npix;
    F = 8 m n for the direct sum (direct / routed / paired / tensor-core paths: the problem's FP32 count,
    whatever unit executes it), 8 m T npix for the bin-count path."""
    path, lanes = srt3d.srt3d_sketch_plan(npix, T, m, n_photons)
    b = 2.0 * n_photons + 4.0 * (npix + 1) + 8.0 * m * npix
    f = 8.0 * m * (T * npix if path == srt3d.PATH_BINCOUNT else n_photons)
    name = {srt3d.PATH_DIRECT: "direct", srt3d.PATH_PAIRED: "paired", srt3d.PATH_ROUTED: "routed",
            srt3d.PATH_TENSOR: "tensor"}.get(path, "bincount")
    return path, lanes, name, b, f


def tc_gemm_flops(npix, T, m):
    """Tensor-core flops one tensor-path sketch launch executes: per pass of M <= 32
    frequencies, a [4 x 32 rows, Kb] x [Kb, 4 MP] f16 GEMM per tile of 4 pixels (MP = 16 if M <= 16
    else 32; Kb = the power of two >= T / 32, at least 16)."""
    q = 4
    while (32 << q) < T:
        q += 1
    f = 0.0
    for j0 in range(0, m, 32):
        mp = 16 if min(32, m - j0) <= 16 else 32
        f += 2.0 * ((npix + 3) // 4 * 4) * 32 * (1 << q) * 4 * mp
    return f


def tensor_roofline(peaks, npix, T, m, ms):
    """The tensor-core sketch against the f16 dense peak (the measured bf16 peak: the same rate)."""
    f = tc_gemm_flops(npix, T, m)
    pk = float(peaks.get("bf16_tflops", 1653.6)) * 1e12
    t = ms * 1e-3
    return {"kernel": "srt3d_sketch (tensor path)", "bound": "tensor", "achieved": f / t / 1e12, "peak": pk / 1e12,
            "unit": "TFLOP/s", "frac": f / pk / t, "executed_tensor_flops_per_launch": f,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (f16 dense: same rate)",
            "note": "tcgen05 kind::f16 histogram x DFT-block GEMM incl. the hi/lo split of V; the kernel is "
                    "bound by shared-memory wavefronts (histogram zeroing + atomics + MMA operand reads: ~97% of "
                    "the 1/clk/SM port in profiles/r02_sketch_tc_ncu_C5.json), not by the tensor pipe"}


def grad_work(npix, m, K, loss=False):
    """Algorithmic bytes / flops of one fused no-loss gradient step: B = 8m + 16K per
    pixel (z, theta in; theta out); F = 21Km + 7m + 3K per pixel minus the |r_j|^2 term (4 per j)
    the no-loss step does not compute."""
    return npix * (8.0 * m + 16.0 * K + (4.0 if loss else 0.0)), npix * (21.0 * K * m + (7.0 if loss else 3.0) * m
                                                                        + 3.0 * K)


def run_sweep(args, torch, srt3d, roofline, s, l2_bytes):
    """Per-config sketch (and gradient) numbers for the workloads SURVEY §8(d) names besides the
    headline: C4@1e6 (the second >= 70 % target: bin-count, HBM-bound), C1-C3 and the C4 sweep.
    Each input is generated, timed and freed in turn."""
    import srt3d_inputs

    flush = (torch.ones(2 * max(l2_bytes, 1 << 20) // 4, dtype=torch.float32, device="cuda"),
             torch.empty(1, dtype=torch.float32, device="cuda"))
    out = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for wl in [w for w in args.sweep_configs.split(",") if w]:
        name, n = (wl.split("@") + [None])[:2]
        n = int(float(n)) if n else None
        t_gen = time.perf_counter()
        fr = srt3d_inputs.make_frame(name, n_per_pixel=n)
        t_gen = time.perf_counter() - t_gen
        bins = torch.from_numpy(fr.bins).cuda()
        offs = torch.from_numpy(fr.offsets).cuda()
        z = torch.empty((fr.npix, fr.m), dtype=torch.complex64, device="cuda")
        path, lanes, pname, b, fl = sketch_work(srt3d, fr.npix, fr.T, fr.m, fr.n_photons)
        small = 2 * fr.n_photons + 8 * fr.m * fr.npix < 2 * l2_bytes  # input + output could stay in L2
        reps = 5 if fr.n_photons > 2e9 else args.sketch_reps
        med, mn = time_sketch(torch, srt3d, bins, offs, z, fr.T, fr.m, fr.n_photons, reps, s,
                              flush if small else None)
        rec = {"workload": fr.name, "npix": fr.npix, "photons": fr.n_photons, "T": fr.T, "m": fr.m,
               "generate_s": round(t_gen, 2),
               "sketch": {"path": pname, "lanes_per_pixel": lanes, "reps": reps, "ms_median": med, "ms_min": mn,
                          "photons_per_s_median": fr.n_photons / (med * 1e-3),
                          "gbs_median": b / (med * 1e-3) / 1e9, "l2": "flushed before every rep" if small else
                          "input larger than L2 (not flushed)",
                          "roofline_median": roofline("srt3d_sketch", b, fl, med),
                          "roofline_min": roofline("srt3d_sketch", b, fl, mn),
                          "roofline_tensor_median": (tensor_roofline(load_peaks()[0], fr.npix, fr.T, fr.m, med)
                                                     if path == srt3d.PATH_TENSOR else None),
                          "traffic": traffic.get(fr.name, {}).get("srt3d_sketch")}}
        if fr.iters:
            t0, a0 = (torch.from_numpy(x).cuda() for x in fr.theta0())
            srt3d.srt3d_sketch(bins, offs, fr.T, fr.m, z=z, total_photons=fr.n_photons, stream=s)
            gb, gf = grad_work(fr.npix, fr.m, fr.K)
            lm, lmin, cm, cmin, cg = time_grad(torch, srt3d, z, t0, a0, fr.sigma, fr.T, fr.m, fr.iters, s, flush)
            rec["grad"] = {"iters_in_graph": fr.iters, "loop_ms_per_iter": lm, "loop_ms_min": lmin,
                           "cold_ms_in_graph": cg, "cold_single_launch_ms_median": cm, "cold_single_launch_ms_min": cmin,
                           "pixel_iters_per_s_loop": fr.npix / (lm * 1e-3),
                           "roofline_cold": roofline("srt3d_sketch_grad_step", gb, gf, cg),
                           "roofline_cold_single_launch": roofline("srt3d_sketch_grad_step", gb, gf, cm),
                           "roofline_loop": roofline("srt3d_sketch_grad_step", gb, gf, lm),
                           "traffic": traffic.get(fr.name, {}).get("srt3d_sketch_grad_step")}
            del t0, a0
        out[fr.name] = rec
        del bins, offs, z, fr
        torch.cuda.empty_cache()
    del flush
    return out


# ------------------------------------------------------------------ GPU arm
def run_srt3d(args):
    import torch
    import torch.distributed as dist

    import paper_2203_00952_b200 as srt3d
    from paper_2203_00952_b200.pipeline import FramePipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    srt3d.load_library()
    f = make_frame(args, rank)
    pipe = FramePipeline(f.n_photons, f.npix, f.K, f.T, f.m, f.sigma, f.iters, fused=not args.unfused,
                         use_graphs=not args.no_graph)
    bins_h = torch.from_numpy(f.bins)
    offs_h = torch.from_numpy(f.offsets)
    t0_h, a0_h = (torch.from_numpy(x) for x in f.theta0())
    pipe.load_device(bins_h, offs_h, t0_h, a0_h)
    pipe.capture()
    s = pipe.stream

    for _ in range(args.warmup):
        pipe.run_device()
    s.synchronize()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(s)
    for k in range(args.steps):
        ev[k][0].record(s)
        pipe.sketch_phase()
        ev[k][1].record(s)
        pipe.iterate_phase()
        ev[k][2].record(s)
    end.record(s)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop() if sampler else None
    ms = start.elapsed_time(end)
    sk_ms = [e[0].elapsed_time(e[1]) for e in ev]
    it_ms = [e[1].elapsed_time(e[2]) for e in ev]
    ms_t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    photons_all = f.n_photons * args.steps * world  # weak scaling: every rank its own frame

    # end-to-end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        bins_p, offs_p = bins_h.pin_memory(), offs_h.pin_memory()
        t0_p, a0_p = t0_h.pin_memory(), a0_h.pin_memory()
        t_out, a_out = torch.empty_like(t0_p).pin_memory(), torch.empty_like(a0_p).pin_memory()
        pipe.run_host(bins_p, offs_p, t0_p, a0_p, t_out, a_out, chunks=args.e2e_chunks)
        pipe.run_host(bins_p, offs_p, t0_p, a0_p, t_out, a_out, chunks=args.e2e_chunks, chain=True)
        s.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for k in range(args.e2e_steps):  # frames stream back to back (chain): PCIe stays busy
            pipe.run_host(bins_p, offs_p, t0_p, a0_p, t_out, a_out, chunks=args.e2e_chunks, chain=k > 0)
        e1.record(s)
        s.synchronize()
        barrier()
        e2e_ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": f.n_photons * args.e2e_steps * world / (float(e2e_ms.item()) * 1e-3), "unit": "photons/s",
               "h2d_bytes_per_step": pipe.h2d_bytes(), "d2h_bytes_per_step": pipe.d2h_bytes(),
               "ms_per_step": float(e2e_ms.item()) / args.e2e_steps, "chunks": args.e2e_chunks,
               "note": "pinned H2D of the frame + theta0, sketch + iterations, D2H of theta, every step; pixel "
                       "blocks pipelined (copy engine uploads block c+1 while block c computes) and frames "
                       "chained (frame f+1's uploads overlap frame f's last block)"}

    # Outside the timed region, on the same buffers: the sketch alone (median / min of
    # --sketch-reps launches) and the gradient step in an `iters`-launch graph and as single
    # launches after an L2 flush (the gradient's roofline fraction uses the
    # L2-cold launch).
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    flush = (torch.ones(2 * max(l2, 1 << 20) // 4, dtype=torch.float32, device="cuda"),
             torch.empty(1, dtype=torch.float32, device="cuda"))
    sk_rep = time_sketch(torch, srt3d, pipe.bins, pipe.offsets, pipe.z, f.T, f.m, f.n_photons, args.sketch_reps, s)
    grad_rep = None
    if f.iters > 0 and pipe.fused:
        grad_rep = time_grad(torch, srt3d, pipe.z, pipe.t0, pipe.a0, f.sigma, f.T, f.m, f.iters, s, flush)
    del flush

    # NEXT-4 streaming acquisition on this frame: the frame's photons as an
    # unsorted event stream (pixel ids shuffled on the GPU) -> CSR, and the
    # count-weighted merge of the frame's sketch into a running sketch.
    stream_ms = None
    if not args.no_stream and f.n_photons < (1 << 31):
        counts = (pipe.offsets[1:].to(torch.int64) - pipe.offsets[:-1].to(torch.int64))
        ev_pix = torch.repeat_interleave(torch.arange(f.npix, device="cuda", dtype=torch.int64), counts)
        perm = torch.randperm(f.n_photons, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7))
        ev_pix = ev_pix[perm].to(torch.int32).view(torch.uint32).contiguous()
        ev_bin = pipe.bins[: f.n_photons].view(torch.int16)[perm].view(torch.uint16).contiguous()
        del perm, counts
        n_run = (pipe.offsets[1:].to(torch.int64) - pipe.offsets[:-1].to(torch.int64)).to(torch.int32).view(
            torch.uint32).contiguous()
        z_run, n_acc = pipe.z.clone(), n_run.clone()
        with torch.cuda.stream(s):
            srt3d.srt3d_bucket_events(ev_pix, ev_bin, f.npix)
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(5)]
            for e in ev:
                e[0].record(s)
                srt3d.srt3d_bucket_events(ev_pix, ev_bin, f.npix)
                e[1].record(s)
                srt3d.srt3d_sketch_merge(z_run, n_acc, pipe.z, n_run, z_out=z_run, n_out=n_acc)
                e[2].record(s)
        s.synchronize()
        stream_ms = {"bucket_ms": statistics.median(e[0].elapsed_time(e[1]) for e in ev),
                     "merge_ms": statistics.median(e[1].elapsed_time(e[2]) for e in ev)}
        del ev_pix, ev_bin, z_run, n_acc, n_run

    # NEXT-2 fused pixelwise fit: the step's `iters` data steps in ONE launch
    # (z staged once, theta in registers; bitwise equal to the iterated steps)
    fit_ms = None
    if f.iters > 0:
        tt, aa = pipe.t0.clone(), pipe.a0.clone()
        with torch.cuda.stream(s):
            srt3d.srt3d_fit_pixelwise(pipe.z, tt, aa, f.sigma, f.T, f.m, f.iters)
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(3)]
            for e in ev:
                tt.copy_(pipe.t0)
                aa.copy_(pipe.a0)
                e[0].record(s)
                srt3d.srt3d_fit_pixelwise(pipe.z, tt, aa, f.sigma, f.T, f.m, f.iters)
                e[1].record(s)
        s.synchronize()
        fit_ms = statistics.median(e[0].elapsed_time(e[1]) for e in ev)

    # NEXT-3 initialisation kernels on this frame's sketch (outside the timed
    # step, which starts from theta0 = t* + 10 per BASELINE.json): greedy
    # backprojection depths (grid N, K picks) and the K = 1 closed form.
    init_ms = None
    if not args.no_init:
        N_grid = min(4096, max(3, args.init_grid or 16 * f.m))
        min_sep = args.init_min_sep
        with torch.cuda.stream(s):
            srt3d.srt3d_init_depths(pipe.z, f.sigma, f.T, N_grid, f.K, min_sep)
            srt3d.srt3d_init_k1(pipe.z, f.sigma, f.T)
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(5)]
            for e in ev:
                e[0].record(s)
                srt3d.srt3d_init_depths(pipe.z, f.sigma, f.T, N_grid, f.K, min_sep)
                e[1].record(s)
                srt3d.srt3d_init_k1(pipe.z, f.sigma, f.T)
                e[2].record(s)
        s.synchronize()
        init_ms = {"N": N_grid, "K": f.K, "min_sep": min_sep,
                   "depths_ms": statistics.median(e[0].elapsed_time(e[1]) for e in ev),
                   "k1_ms": statistics.median(e[1].elapsed_time(e[2]) for e in ev)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks, peak_kind = load_peaks()
    hbm = float(peaks.get("hbm_gbs", 6547.8))
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    fp32_peak = nsm * FP32_LANES_PER_SM * 2 * sm_max * 1e6  # flop/s at max clock
    sk_avg = statistics.mean(sk_ms)
    it_avg = statistics.mean(it_ms)
    peak_src_fp32 = f"FP32: {nsm} SMs x 128 lanes x 2 flop x {sm_max:.0f} MHz (max clock; unit-count derivation)"
    peak_src_hbm = f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"

    def roofline(kernel, bytes_, flops, ms):
        """t_roof = max(bytes / HBM peak, flops / FP32 peak); frac = t_roof / t_measured."""
        t_hbm, t_fp32 = bytes_ / (hbm * 1e9), flops / fp32_peak
        t = ms * 1e-3
        if t_hbm >= t_fp32:
            return {"kernel": kernel, "bound": "hbm", "achieved": bytes_ / t / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": t_hbm / t, "peak_source": peak_src_hbm, "alg_bytes_per_launch": bytes_,
                    "alg_flops_per_launch": flops}
        return {"kernel": kernel, "bound": "alu", "achieved": flops / t / 1e12, "peak": fp32_peak / 1e12,
                "unit": "TFLOP/s", "frac": t_fp32 / t, "peak_source": peak_src_fp32, "alg_bytes_per_launch": bytes_,
                "alg_flops_per_launch": flops}

    # sketch: B = 2n + 4(npix+1) + 8 m npix bytes; F = 8 m n (direct) or 8 m T npix (bin-count)
    path, lanes, pname, sk_bytes, sk_flops = sketch_work(srt3d, f.npix, f.T, f.m, f.n_photons)
    try:
        fp32_meas = srt3d.srt3d_debug_ffma_peak() * 1e12  # K8, measured in this run
    except Exception:  # pragma: no cover - measurement utility only
        fp32_meas = None
    sketch = {"kernel": "srt3d_sketch", "path": pname, "lanes_per_pixel": lanes, "ms": sk_avg,
              "ms_in_step_per_rep": sk_ms, "ms_median": sk_rep[0], "ms_min": sk_rep[1], "reps": args.sketch_reps,
              "photons_per_s": f.n_photons / (sk_avg * 1e-3),
              "gbs": sk_bytes / (sk_avg * 1e-3) / 1e9, "frac_hbm": (sk_bytes / (sk_avg * 1e-3) / 1e9) / hbm,
              "tflops_direct_count": 8.0 * f.m * f.n_photons / (sk_avg * 1e-3) / 1e12,
              "roofline": roofline("srt3d_sketch", sk_bytes, sk_flops, sk_avg),
              "roofline_median": roofline("srt3d_sketch", sk_bytes, sk_flops, sk_rep[0]),
              "roofline_min": roofline("srt3d_sketch", sk_bytes, sk_flops, sk_rep[1]),
              "fp32_measured_tflops": fp32_meas / 1e12 if fp32_meas else None,
              "frac_of_measured_fp32": (sk_flops / (sk_avg * 1e-3)) / fp32_meas if fp32_meas else None}
    if path == srt3d.PATH_TENSOR:
        sketch["roofline_tensor"] = tensor_roofline(peaks, f.npix, f.T, f.m, sk_avg)
        sketch["roofline_note"] = ("roofline: the north-star definition (slower of bytes at HBM peak and the direct "
                                   "sum's 8 m n flops at FP32 peak); above 1 because the tensor-core path evaluates "
                                   "the sum as a GEMM on the binned photons; roofline_tensor: the executed GEMM vs "
                                   "the f16 tensor peak")
    grad = None
    if f.iters > 0:
        per_iter = it_avg / f.iters
        g_bytes, g_flops = grad_work(f.npix, f.m, f.K)
        if not pipe.fused:  # grad (with loss buffer untouched: NL) + separate update: theta read twice, grads through HBM
            g_bytes = f.npix * (8.0 * f.m + 32.0 * f.K + 16.0 * f.K)
        kname = "srt3d_sketch_grad_step" if pipe.fused else "srt3d_sketch_grad+srt3d_descent_update"
        grad = {"kernel": kname, "ms_per_iter": per_iter, "pixel_iters_per_s": f.npix / (per_iter * 1e-3),
                "gbs": g_bytes / (per_iter * 1e-3) / 1e9, "tflops": g_flops / (per_iter * 1e-3) / 1e12,
                "alg_work": "per pixel-iteration B = 8m + 16K bytes, F = 21Km + 3m + 3K flops (no-loss fused step: "
                            "the |r|^2 term of SURVEY §8(d)'s 21Km + 7m + 3K is not computed)",
                "roofline_in_loop": roofline(kname, g_bytes, g_flops, per_iter),
                "note": "in-loop (CUDA-graph) time per iteration incl. node launch gaps; theta stays L2-resident "
                        "across iterations and z (67 MB) partly: the same loop alternating two copies of z "
                        "(134 MB > L2, z always from HBM) runs 14.7 instead of 13.6 us per iteration "
                        "(tools/grad_probe.py loop_two_z_us_median)"}
        if grad_rep is not None:
            grad.update({"loop_graph_ms_per_iter": grad_rep[0], "cold_l2_ms_per_launch": grad_rep[4],
                         "cold_l2_single_launch_ms_median": grad_rep[2], "cold_l2_single_launch_ms_min": grad_rep[3],
                         "cold_l2_note": "every launch after an L2 flush that READS 2x L2 (clean lines). "
                                         "cold_l2_ms_per_launch: CUDA events around graphs of 20 x [flush, step] minus "
                                         "20 x [flush] (the kernel without its launch latency; ncu's "
                                         "gpu__time_duration of the same launch agrees); single_launch: events "
                                         "around one launch (adds ~2.5 us of launch latency), median / min of 20",
                         "roofline": roofline(kname, g_bytes, g_flops, grad_rep[4]),
                         "roofline_cold_single_launch": roofline(kname, g_bytes, g_flops, grad_rep[2])})
        else:
            grad["roofline"] = grad["roofline_in_loop"]
    init = None
    if init_ms is not None:
        # backprojection + picks: F = 8 m N per pixel (one complex multiply-add per (grid point, l));
        # B = 8 m + 12 K + 4 per pixel.  K = 1 closed form: B = 8 m + 8, F = 8 m per pixel (phasor
        # step + weighted real part), HBM-bound.
        d_b = f.npix * (8.0 * f.m + 12.0 * f.K + 4.0)
        d_f = f.npix * 8.0 * f.m * init_ms["N"]
        k_b = f.npix * (8.0 * f.m + 8.0)
        k_f = f.npix * 8.0 * f.m
        n_grid = init_ms["N"]
        tc_path = n_grid % 32 == 0 and 32 <= n_grid <= 512 and f.m <= 32  # init_tc.cu shapes
        if tc_path:
            # tensor-core path: the backprojection is the GEMM [Re z, Im z] (npix x 2m) x B^T (2m x N);
            # algorithmic flops 2 (2m) N per pixel (the hi/lo split executes 3x that); TF32 dense peak =
            # the measured bf16 peak x 1.1/2.25 (B200_PROFILING.md nominal ratio)
            bf16 = float(peaks.get("bf16_tflops", 1653.6)) * 1e12
            tf32_peak = bf16 * 1.1 / 2.25
            t_alg = f.npix * 2.0 * (2.0 * f.m) * n_grid
            t_run = init_ms["depths_ms"] * 1e-3
            d_roof = {"kernel": "srt3d_init_depths", "bound": "tensor", "achieved": t_alg / t_run / 1e12,
                      "peak": tf32_peak / 1e12, "unit": "TFLOP/s", "frac": t_alg / tf32_peak / t_run,
                      "peak_source": "MEASURED_PEAKS.json bf16_tflops x 1.1/2.25 (TF32 dense)",
                      "alg_flops_per_launch": t_alg, "executed_tensor_flops_per_launch": 3.0 * f.npix * 2.0 * 64 * n_grid,
                      "note": "tcgen05 kind::tf32 (3-term split) + pick epilogue; the next tile's MMAs run under "
                              "the current tile's pick rounds, and the TMEM candidate scan (~6 instructions per grid "
                              "point) bounds the kernel (profiles/r02_init_depths_ncu_C5.json, DESIGN.md 5.5)"}
        else:
            d_roof = roofline("srt3d_init_depths", d_b, d_f, init_ms["depths_ms"])
        init = {"init_depths": {"kernel": "srt3d_init_depths", "grid_N": init_ms["N"], "K": init_ms["K"],
                                "min_sep": init_ms["min_sep"], "ms": init_ms["depths_ms"],
                                "path": "tensor cores (tcgen05)" if tc_path else "cuda cores",
                                "pixels_per_s": f.npix / (init_ms["depths_ms"] * 1e-3),
                                "roofline": d_roof},
                "init_k1": {"kernel": "srt3d_init_k1", "ms": init_ms["k1_ms"],
                            "pixels_per_s": f.npix / (init_ms["k1_ms"] * 1e-3),
                            "roofline": roofline("srt3d_init_k1", k_b, k_f, init_ms["k1_ms"])},
                "note": "NEXT-3, timed outside the step (the step starts from theta0 = t* + 10)"}
    fit = None
    if fit_ms is not None:
        # same arithmetic per pixel-iteration as the step (F below); bytes: z and theta once per launch
        f_f = f.iters * f.npix * (21.0 * f.K * f.m + 7.0 * f.m + 3.0 * f.K)
        f_b = f.npix * (8.0 * f.m + 16.0 * f.K)
        fit = {"kernel": "srt3d_fit_pixelwise", "iters": f.iters, "ms": fit_ms,
               "pixel_iters_per_s": f.npix * f.iters / (fit_ms * 1e-3),
               "roofline": roofline("srt3d_fit_pixelwise", f_b, f_f, fit_ms),
               "note": "NEXT-2: the iterations of the step in one launch (no spatial regulariser between data "
                       "steps); bitwise equal to iters x srt3d_sketch_grad_step; timed outside the step",
               # the same step (identical theta) with the iterations fused: sketch + one fit launch
               "step_with_fused_iterations": {"ms": sk_avg + fit_ms, "unit": "photons/s",
                                              "value": f.n_photons * world / ((sk_avg + fit_ms) * 1e-3)}}
    stream = None
    if stream_ms is not None:
        # bucketing: read each (uint32 pixel, uint16 bin) event once, write its bin, write offsets
        b_b = 8.0 * f.n_photons + 4.0 * (f.npix + 1)
        # merge: read two sketch rows + counts, write one
        m_b = f.npix * (3 * 8.0 * f.m + 3 * 4.0)
        stream = {"bucket_events": {"kernel": "srt3d_bucket_events", "events": f.n_photons, "ms": stream_ms["bucket_ms"],
                                    "events_per_s": f.n_photons / (stream_ms["bucket_ms"] * 1e-3),
                                    "roofline": roofline("srt3d_bucket_events", b_b, 0.0, stream_ms["bucket_ms"]),
                                    "note": "two-level counting sort (coarse histogram, bucket partition, per-bucket tile sort); algorithmic 8 B/event (read 6, write 2), design traffic 24 B/event (DESIGN.md §5.6)"},
                  "sketch_merge": {"kernel": "srt3d_sketch_merge", "ms": stream_ms["merge_ms"],
                                   "roofline": roofline("srt3d_sketch_merge", m_b, 0.0, stream_ms["merge_ms"])},
                  "note": "NEXT-4, timed outside the step"}
    # dominant kernel (larger share of the step) -> the line's roofline object.  The gradient's
    # headline fraction is its L2-cold launch; the in-loop fraction rides along.
    # `traffic` is the DRAM bytes per launch of an ncu --set full capture of the same kernel and
    # config (profiles/traffic.json; a captured profile, not this run: ncu cannot run inside the bench).
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(f.name, {})
    if grad is None or sk_avg >= it_avg:
        roof = dict(sketch["roofline"])
        roof["traffic"] = traffic.get("srt3d_sketch")
        roof["share_of_step"] = sk_avg / (sk_avg + it_avg)
    else:
        roof = dict(grad["roofline"])
        roof["traffic"] = traffic.get("srt3d_sketch_grad_step")
        roof["share_of_step"] = it_avg / (sk_avg + it_avg)
        roof["frac_in_loop"] = grad["roofline_in_loop"]["frac"]
        roof["timing"] = ("frac: L2-cold launch (events around graphs of [L2 flush, step] minus [L2 flush]); "
                          "frac_in_loop: per iteration of the step")
    roof["traffic_source"] = "profiles/traffic.json (ncu --set full capture, DRAM read+write bytes per launch)"
    launches = pipe.launches_per_step * args.steps
    sweep = None
    if not args.no_sweep and world == 1:
        del pipe  # free the headline frame's buffers (the C4@1e6 input alone is 8.2 GB)
        torch.cuda.empty_cache()
        sweep = run_sweep(args, torch, srt3d, roofline, torch.cuda.Stream(), l2)

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        info = oracle_step_sample(f, args.cpu_seconds, single_core=True)
        cpu = {"value": info["photons"] / info["seconds"], "unit": "photons/s", "cores": info["cores"],
               "kind": "oracle", "sample": info["sample"], "cpu_model": info["cpu_model"],
               "one_core": info.get("one_core")}

    line = {"metric": METRIC, "value": photons_all / (ms_max * 1e-3), "unit": "photons/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Eq. (1) photon frames; stand-in for the paper's head/camouflage datasets)",
            "config": config_obj(f, args), "clocks": clocks, "e2e": e2e,
            "gpu_launches": launches,
            "roofline": roof, "cpu_baseline": cpu, "sketch": sketch, "grad": grad, "fit": fit, "init": init,
            "stream": stream, "sweep": sweep,
            "step_definition": "srt3d_sketch over the frame + iters x srt3d_sketch_grad_step (CUDA graphs)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_srt3d(args)


if __name__ == "__main__":
    sys.exit(main())
