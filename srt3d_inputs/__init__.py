"""Seeded synthetic inputs for the SRT3D hot path (shared by oracle tests, GPU
tests and bench.py).  Holds no part of the method's arithmetic: it only
builds scenes and samples photon time stamps from the Eq. (1) mixture
 with the native sampler in ``gen.c``.

The five presets follow BASELINE.json ``configs[0..4]`` (C1..C5) with the
specifics SURVEY.md §8(d) proposes (see DESIGN.md §4 "Input recipe"):

  intensity model (reading A9): background mean b = lam/(1+SBR) per pixel,
  signal mean lam_ik = lam*SBR/(1+SBR) * a_ik / mean_i(sum_k a_ik),
  n_i ~ Poisson(b + sum_k lam_ik), true alpha_ik = lam_ik / (b + sum_k lam_ik).
  Absent (padded) surfaces: alpha = 0, t = t_1 + T/2 (reading A14).
  Initial depth for the fit: t0 = t* + 10 bins, alpha0 = alpha* (reading A13).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsrt3d_gen.so")
_lib = None


def build(force: bool = False) -> str:
    import subprocess

    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        lib.srt3d_gen_counts.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, P]
        lib.srt3d_gen_photons.argtypes = [P, ctypes.c_int64, ctypes.c_uint32, P, P, ctypes.c_double,
                                          ctypes.c_uint32, ctypes.c_uint64, P]
        lib.srt3d_gen_counts.restype = ctypes.c_int
        lib.srt3d_gen_photons.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def sample_photons(t, weights, sigma: float, T: int, seed: int, mean=None, fixed_n: int | None = None,
                   offsets_dtype=np.uint32):
    """Sample a pixel-sorted CSR photon frame.

    t: float32 (npix, K) depths; weights: float64 (npix, K+1) = (b, lam_1..lam_K)
    relative class weights; mean: float64 (npix,) Poisson means, or fixed_n.
    Returns (bins uint16 [N], offsets uint32 [npix+1])."""
    t = np.ascontiguousarray(t, dtype=np.float32)
    npix, K = t.shape
    weights = np.ascontiguousarray(weights, dtype=np.float64).reshape(npix, K + 1)
    counts = np.zeros(npix, dtype=np.uint64)
    if fixed_n is not None:
        mean_arr = np.zeros(1, dtype=np.float64)
        _load().srt3d_gen_counts(_p(mean_arr), npix, int(fixed_n), int(seed) & (2**64 - 1), _p(counts))
    else:
        mean_arr = np.ascontiguousarray(mean, dtype=np.float64)
        _load().srt3d_gen_counts(_p(mean_arr), npix, -1, int(seed) & (2**64 - 1), _p(counts))
    off64 = np.zeros(npix + 1, dtype=np.uint64)
    np.cumsum(counts, out=off64[1:])
    total = int(off64[-1])
    if total >= 2**32:
        raise ValueError("frame exceeds 2^32 photons (uint32 CSR offsets)")
    offsets = off64.astype(offsets_dtype)
    bins = np.empty(total, dtype=np.uint16)
    rc = _load().srt3d_gen_photons(_p(offsets), npix, K, _p(weights), _p(t), float(sigma), int(T),
                                   int(seed) & (2**64 - 1), _p(bins))
    if rc != 0:
        raise RuntimeError(f"srt3d_gen_photons failed ({rc})")
    return bins, offsets


@dataclass
class Frame:
    name: str
    rows: int
    cols: int
    T: int
    m: int
    K: int
    sigma: float
    iters: int
    lam: float
    sbr: float
    seed: int
    bins: np.ndarray
    offsets: np.ndarray
    t_true: np.ndarray  # float32 (npix, K)
    alpha_true: np.ndarray  # float32 (npix, K)
    recipe: dict = field(default_factory=dict)

    @property
    def npix(self) -> int:
        return self.rows * self.cols

    @property
    def n_photons(self) -> int:
        return int(self.offsets[-1]) - int(self.offsets[0])

    def theta0(self):
        """Initial fit state (reading A13): t0 = t* + 10 bins, alpha0 = alpha*."""
        t0 = (self.t_true + np.float32(10.0)).astype(np.float32)
        return t0, self.alpha_true.copy()


CONFIGS = {
    "C1": dict(rows=32, cols=32, T=1024, sigma=2.0, lam=50.0, sbr=1.0, m=4, K=1, iters=20, seed=101),
    "C2": dict(rows=141, cols=141, T=4613, sigma=5.0, lam=1000.0, sbr=1.0, m=10, K=1, iters=100, seed=102),
    "C3": dict(rows=256, cols=256, T=2500, sigma=3.0, lam=10000.0, sbr=0.1, m=20, K=2, iters=100, seed=103),
    "C4": dict(rows=64, cols=64, T=4096, sigma=4.0, lam=None, sbr=1.0, m=10, K=1, iters=0, seed=104),
    "C5": dict(rows=512, cols=512, T=8192, sigma=6.0, lam=1000.0, sbr=0.01, m=32, K=3, iters=200, seed=105),
}
C4_SWEEP = [100, 1000, 10000, 100000, 1000000]


def _scene(name: str, rows: int, cols: int, T: int, K: int, rng: np.random.Generator):
    """Per-pixel depths t (npix, K) and relative intensities a (npix, K)."""
    r, c = np.meshgrid(np.arange(rows, dtype=np.float64), np.arange(cols, dtype=np.float64), indexing="ij")
    npix = rows * cols
    if name == "C1":  # tilted plane spanning 300..700 (BASELINE configs[0])
        t = (300.0 + 400.0 * (r + c) / (rows + cols - 2)).reshape(npix, 1)
        a = rng.uniform(0.5, 1.0, size=(npix, 1))
    elif name == "C2":  # smooth sum of 8 Gaussian bumps mapped onto 1000..3500 (configs[1])
        surf = np.zeros_like(r)
        for _ in range(8):
            A = rng.uniform(0.5, 1.0)
            cr, cc = rng.uniform(0, rows), rng.uniform(0, cols)
            s = rng.uniform(8.0, 30.0)
            surf += A * np.exp(-((r - cr) ** 2 + (c - cc) ** 2) / (2 * s * s))
        lo, hi = surf.min(), surf.max()
        t = (1000.0 + 2500.0 * (surf - lo) / max(hi - lo, 1e-12)).reshape(npix, 1)
        a = rng.uniform(0.2, 1.0, size=(npix, 1))
    elif name == "C3":  # foreground rectangle occluding a background plane (configs[2])
        back = 1600.0 + 400.0 * c / (cols - 1)
        fg = (c >= cols // 4) & (c < 3 * cols // 4)  # columns 64..191: exactly half the pixels
        t = np.zeros((npix, 2))
        a = np.zeros((npix, 2))
        fgf = fg.reshape(-1)
        t[:, 0] = np.where(fgf, 800.0, back.reshape(-1))
        t[:, 1] = np.where(fgf, back.reshape(-1), back.reshape(-1) + T / 2.0)
        a[:, 0] = np.where(fgf, 0.5, 1.0)
        a[:, 1] = np.where(fgf, 0.5, 0.0)
    elif name == "C4":  # one surface at a uniformly random real depth (configs[3])
        t = rng.uniform(0.0, float(T), size=(npix, 1))
        a = np.ones((npix, 1))
    elif name == "C5":  # 3 depths, circular gaps >= 50 bins (configs[4])
        t = np.zeros((npix, 3))
        for i in range(npix):
            while True:
                d = np.sort(rng.uniform(0.0, float(T), size=3))
                gaps = np.diff(np.concatenate([d, [d[0] + T]]))
                if gaps.min() >= 50.0:
                    break
            t[i] = d
        a = rng.uniform(0.05, 1.0, size=(npix, 3))
    else:
        raise KeyError(name)
    t = np.mod(t, float(T))
    return t, a


def _scene_c5_fast(npix: int, T: int, rng: np.random.Generator):
    """Vectorised rejection sampler for C5 depths (same law as the loop)."""
    out = np.zeros((npix, 3))
    todo = np.arange(npix)
    while todo.size:
        d = np.sort(rng.uniform(0.0, float(T), size=(todo.size, 3)), axis=1)
        gaps = np.diff(np.concatenate([d, d[:, :1] + T], axis=1), axis=1)
        ok = gaps.min(axis=1) >= 50.0
        out[todo[ok]] = d[ok]
        todo = todo[~ok]
    return out


def make_frame(name: str, n_per_pixel: int | None = None, seed: int | None = None,
               rows: int | None = None, cols: int | None = None) -> Frame:
    """Build config ``name`` ('C1'..'C5'); for C4 give ``n_per_pixel``.

    ``rows``/``cols`` may shrink a preset (same recipe, fewer pixels) for
    quick tests."""
    cfg = dict(CONFIGS[name])
    if seed is None:
        seed = cfg["seed"] + (C4_SWEEP.index(n_per_pixel) if (name == "C4" and n_per_pixel in C4_SWEEP) else 0)
    rows = rows or cfg["rows"]
    cols = cols or cfg["cols"]
    T, K, sigma, sbr = cfg["T"], cfg["K"], cfg["sigma"], cfg["sbr"]
    rng = np.random.default_rng(seed)
    npix = rows * cols
    if name == "C5":
        t = _scene_c5_fast(npix, T, rng)
        a = rng.uniform(0.05, 1.0, size=(npix, 3))
    else:
        t, a = _scene(name, rows, cols, T, K, rng)
    recipe = {"scene": name, "rows": rows, "cols": cols, "T": T, "K": K, "sigma": sigma, "SBR": sbr,
              "seed": seed, "m": cfg["m"], "iters": cfg["iters"],
              "intensity_model": "A9: b=lam/(1+SBR); lam_k=lam*SBR/(1+SBR)*a_k/mean(sum a)",
              "signal_law": "wrapped discrete Gaussian (A8)"}
    if name == "C4":
        if n_per_pixel is None:
            raise ValueError("C4 needs n_per_pixel")
        # each photon is signal with probability SBR/(1+SBR) = 0.5
        weights = np.stack([np.full(npix, 1.0 / (1 + sbr)), np.full(npix, sbr / (1 + sbr))], axis=1)
        bins, offsets = sample_photons(t.astype(np.float32), weights, sigma, T, seed, fixed_n=n_per_pixel)
        alpha = np.full((npix, 1), sbr / (1 + sbr))
        lam = float(n_per_pixel)
        recipe["photons_per_pixel"] = n_per_pixel
    else:
        lam = cfg["lam"]
        b = lam / (1.0 + sbr)
        abar = a.sum(axis=1).mean()
        lam_k = lam * sbr / (1.0 + sbr) * a / abar
        mean = b + lam_k.sum(axis=1)
        weights = np.concatenate([np.full((npix, 1), b), lam_k], axis=1)
        bins, offsets = sample_photons(t.astype(np.float32), weights, sigma, T, seed, mean=mean)
        alpha = lam_k / mean[:, None]
        recipe["lambda"] = lam
    return Frame(name=name if name != "C4" else f"C4@{n_per_pixel:.0e}".replace("+0", ""), rows=rows, cols=cols,
                 T=T, m=cfg["m"], K=K, sigma=sigma, iters=cfg["iters"], lam=lam, sbr=sbr, seed=seed,
                 bins=bins, offsets=offsets, t_true=t.astype(np.float32), alpha_true=alpha.astype(np.float32),
                 recipe=recipe)


def random_csr(npix: int, T: int, max_n: int, seed: int, empty_frac: float = 0.1):
    """Ragged random CSR frame for edge-case tests: per-pixel counts uniform in
    [0, max_n] (a fraction of them forced empty), uniform stamps on {0..T-1}."""
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, max_n + 1, size=npix)
    counts[rng.random(npix) < empty_frac] = 0
    offsets = np.zeros(npix + 1, dtype=np.uint64)
    np.cumsum(counts, out=offsets[1:])
    bins = rng.integers(0, T, size=int(offsets[-1]), dtype=np.int64).astype(np.uint16)
    return bins, offsets.astype(np.uint32)


def random_theta(npix: int, K: int, T: int, seed: int, alpha_lo: float = 0.0, alpha_hi: float = 1.0):
    """Random fp32 parameters: t uniform on [0, T), alpha uniform on [lo, hi]."""
    rng = np.random.default_rng(seed)
    t = rng.uniform(0.0, float(T), size=(npix, K)).astype(np.float32)
    a = rng.uniform(alpha_lo, alpha_hi, size=(npix, K)).astype(np.float32)
    return t, a


def random_sketch(npix: int, m: int, seed: int, scale: float = 0.5):
    """Random complex64 sketch-shaped array with |z| <= ~scale."""
    rng = np.random.default_rng(seed)
    return (scale * (rng.uniform(-1, 1, size=(npix, m)) + 1j * rng.uniform(-1, 1, size=(npix, m)))).astype(np.complex64)
