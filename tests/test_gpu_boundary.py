"""The C-ABI boundary contract (include/srt3d.h conventions), on the GPU:

  * srt3d_sketch(bins, offsets, npix, T, m, z, stream) picks its launch regime on the
    device — no host read, no synchronisation — so it is CUDA-graph capturable, and the
    regime follows the photon counts present in device memory at replay time;
  * the hint-less call gives bitwise the result of the hinted call (same kernel selected)
    for frames in every regime, and matches the oracle (Eq. (3));
  * bins >= T (a precondition violation) give finite values and never fault, on every path;
  * calls are reentrant: two host threads on two streams get bitwise the serial results.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SKETCH_ATOL = 1e-5


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _fixed_csr(npix, n, T, seed):
    rng = np.random.default_rng(seed)
    counts = rng.integers(max(1, n - n // 8), n + n // 8 + 1, npix)
    counts[::17] = 0  # empty pixels
    offs = np.zeros(npix + 1, np.uint32)
    offs[1:] = np.cumsum(counts)
    bins = rng.integers(0, T, int(offs[-1])).astype(np.uint16)
    return bins, offs


# (T, m, mean photons per pixel, npix) -> one frame per regime of sketch_regime():
# G4 (< 256), G8 (256..2047, M < 24), RT (256..2047, M >= 24, T % 4 == 0, T <= 12000), G4C (the
# same where RT does not apply: odd T here, and the second pass of m = 60), G16 (2048..4095),
# G32 (>= 4096, below T), bin-count with 128 / 256 / 512 threads (>= T; < 3e4, < 8e4, more)
REGIME_FRAMES = [(8192, 10, 60, 600), (8192, 10, 700, 300), (8192, 32, 700, 300), (4613, 32, 700, 300),
                 (8192, 60, 700, 100), (8192, 32, 2600, 100),
                 (8192, 40, 5000, 60), (1024, 10, 4000, 60), (1024, 4, 40000, 24), (1024, 20, 90000, 12)]


@pytest.mark.parametrize("T,m,n,npix", REGIME_FRAMES)
def test_hintless_sketch_equals_hinted_and_oracle(gpu, oracle_mod, T, m, n, npix):
    import torch

    bins, offs = _fixed_csr(npix, n, T, seed=T + m + n)
    db, do = _dev(bins), _dev(offs)
    z_dev = gpu.srt3d_sketch(db, do, T, m)                                # C srt3d_sketch, no hint
    z_hint = gpu.srt3d_sketch(db, do, T, m, total_photons=int(offs[-1]))  # srt3d_sketch_ex with the hint
    torch.cuda.synchronize()
    assert torch.equal(z_dev.view(torch.float32), z_hint.view(torch.float32)), "device-selected regime differs"
    zo = oracle_mod.sketch(bins, offs, T, m)
    d = np.abs(z_dev.cpu().numpy() - zo)
    assert max(np.abs(d.real).max(), np.abs(d.imag).max()) <= SKETCH_ATOL


def test_hintless_sketch_in_cuda_graph_follows_device_data(gpu, oracle_mod):
    """Capture srt3d_sketch once (frame A resident), then overwrite the device buffers with
    frames of other regimes (B: ~3000 photons/pixel, C: ~20000 photons/pixel, bin-count)
    and replay: each replay equals the oracle sketch of the data present at replay time."""
    import torch

    T, m, npix = 4096, 32, 96
    frames = [_fixed_csr(npix, n, T, seed=n) for n in (40, 3000, 20000)]
    cap = max(int(o[-1]) for _, o in frames)
    db = torch.zeros(cap, dtype=torch.uint16, device="cuda")
    do = torch.zeros(npix + 1, dtype=torch.uint32, device="cuda")
    z = torch.zeros((npix, m), dtype=torch.complex64, device="cuda")

    def load(k):
        b, o = frames[k]
        db[: len(b)].copy_(_dev(b))
        do.copy_(_dev(o))

    load(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        gpu.srt3d_sketch(db, do, T, m, z=z)  # warm-up outside capture (attributes, caches)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        gpu.srt3d_sketch(db, do, T, m, z=z)
    for k in (1, 2, 0):
        load(k)
        z.zero_()
        g.replay()
        torch.cuda.synchronize()
        b, o = frames[k]
        zo = oracle_mod.sketch(b, o, T, m)
        d = z.cpu().numpy() - zo
        assert max(np.abs(d.real).max(), np.abs(d.imag).max()) <= SKETCH_ATOL, k


@pytest.mark.parametrize("T", [1000, 8192])
def test_out_of_range_bins_finite_on_every_path(gpu, oracle_mod, T):
    """bins >= T violate the precondition: every path must still return OK, write finite
    values everywhere, and leave the pixels without bad bins exact (no memory corruption)."""
    import torch

    rng = np.random.default_rng(T)
    npix, n = 64, 3000
    bins, offs = _fixed_csr(npix, n, T, seed=5)
    bad_pix = np.arange(0, npix, 5)
    for i in bad_pix:  # sprinkle out-of-range bins, including the maximum 65535
        b0, b1 = int(offs[i]), int(offs[i + 1])
        if b1 > b0:
            k = rng.integers(b0, b1, max(1, (b1 - b0) // 10))
            bins[k] = rng.integers(T, 65536, k.size).astype(np.uint16)
            bins[b0] = 65535
    good = np.setdiff1d(np.arange(npix), bad_pix)
    sel = np.concatenate([[0], np.cumsum(np.diff(offs.astype(np.int64))[good])]).astype(np.uint32)
    gbins = np.concatenate([bins[offs[i]:offs[i + 1]] for i in good])
    zo = oracle_mod.sketch(gbins, sel, T, 32)
    db, do = _dev(bins), _dev(offs)
    calls = [dict(), dict(total_photons=int(offs[-1]))]
    calls += [dict(path=gpu.PATH_DIRECT, lanes_per_pixel=g, total_photons=int(offs[-1])) for g in (4, 8, 16, 32)]
    calls += [dict(path=gpu.PATH_BINCOUNT), dict(path=gpu.PATH_PAIRED), dict(path=gpu.PATH_DIRECT),
              dict(path=gpu.PATH_ROUTED), dict(path=gpu.PATH_ROUTED, lanes_per_pixel=2), dict(path=gpu.PATH_TENSOR)]
    for kw in calls:
        if "path" in kw:
            z = gpu.srt3d_sketch_ex(db, do, T, 32, **kw)
        else:
            z = gpu.srt3d_sketch(db, do, T, 32, **kw)
        torch.cuda.synchronize()
        zh = z.cpu().numpy()
        assert np.all(np.isfinite(zh.view(np.float32))), kw
        d = zh[good] - zo
        assert max(np.abs(d.real).max(), np.abs(d.imag).max()) <= SKETCH_ATOL, kw


def _workload(gpu, inputs_mod, seed, stream):
    """A mix of entry points on one stream: sketch (device regime), expected sketch,
    gradient, fused steps, init, merge."""
    import torch

    T, m, K, sigma = 8192, 32, 3, 6.0
    bins, offs = _fixed_csr(500, 900, T, seed=seed)
    t, a = inputs_mod.random_theta(500, K, T, seed=seed)
    with torch.cuda.stream(stream):
        db, do, dt, da = _dev(bins), _dev(offs), _dev(t), _dev(a)
        outs = []
        for _ in range(4):
            z = gpu.srt3d_sketch(db, do, T, m, stream=stream)
            phi = gpu.srt3d_expected_sketch(dt, da, sigma, T, m, stream=stream)
            gt, ga, L = gpu.srt3d_sketch_grad(z, dt, da, sigma, T, m, stream=stream)
            t1, a1 = dt.clone(), da.clone()
            for _ in range(3):
                gpu.srt3d_sketch_grad_step(z, t1, a1, sigma, T, m, 0.5, stream=stream)
            ti, gi, ai, ci = gpu.srt3d_init_depths(z, sigma, T, 512, K, 50, stream=stream)
            outs.append([x.clone() for x in (z, phi, gt, ga, L, t1, a1, ti, ci)])
    stream.synchronize()
    return outs


def test_reentrant_two_threads_two_streams(gpu, inputs_mod):
    """No global mutable state (SURVEY §8(b) conventions): two host threads driving the
    library concurrently on two streams get bitwise the single-threaded results."""
    import torch

    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    ref = [_workload(gpu, inputs_mod, seed, s0) for seed in (1, 2)]
    res = [None, None]
    errs = []

    def run(k, stream):
        try:
            torch.cuda.set_device(0)
            res[k] = _workload(gpu, inputs_mod, k + 1, stream)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(k, s)) for k, s in ((0, s0), (1, s1))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for k in range(2):
        for it_ref, it_res in zip(ref[k], res[k]):
            for u, v in zip(it_ref, it_res):
                assert torch.equal(u.view(torch.uint8), v.view(torch.uint8))


_PDL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2203_00952_b200 as p
from paper_2203_00952_b200.pipeline import FramePipeline  # noqa: F401  (same package state as the bench)
g = torch.Generator(device="cuda").manual_seed(3)
npix, m, K, T, sigma = 70001, 32, 3, 8192, 6.0
t = torch.rand((npix, K), device="cuda", generator=g) * T
a = torch.rand((npix, K), device="cuda", generator=g)
z = torch.randn((npix, m), dtype=torch.complex64, device="cuda", generator=g)
s = torch.cuda.Stream()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=s):
    for _ in range(7):
        p.srt3d_sketch_grad_step(z, t, a, sigma, T, m, 0.5, stream=s)
graph.replay()
for _ in range(3):  # and as ordinary stream launches behind other kernels
    z.mul_(1.0)
    p.srt3d_sketch_grad_step(z, t, a, sigma, T, m, 0.5)
torch.cuda.synchronize()
np.save(sys.argv[2], np.concatenate([t.cpu().numpy().ravel(), a.cpu().numpy().ravel()]))
"""


def test_programmatic_dependent_launch_bitwise(tmp_path):
    """The TMA gradient step is launched as a programmatic dependent (griddepcontrol.wait before
    any global read): graph-replayed and stream-ordered steps give bitwise the
    theta of ordinary launches (SRT3D_PDL=0)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = tmp_path / f"theta_{flag}.npy"
        env = dict(os.environ, SRT3D_PDL=flag)
        r = subprocess.run([sys.executable, "-c", _PDL_SCRIPT, root, str(out)], env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
