"""ORACLE — test infrastructure only.

Plain fp64 CPU implementation of the SRT3D hot path (Eq. (3), (4),
(6)/(8)), in ``oracle/srt3d_ref.c``, loaded through ctypes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` and
``--impl reference``) may import this package.  It shares no code with the
CUDA path in ``paper_2203_00952_b200/`` and imports nothing from it.

Every function here is pinned by ``tests/test_oracle_pins.py`` (closed forms,
special cases, brute force, finite differences); there is no "parity
unpinned" function.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/srt3d_ref.c with gcc (plain -O2, no fast-math)."""
    import subprocess

    src = os.path.join(_HERE, "srt3d_ref.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"]
        )
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, u32, f64, i32 = ctypes.c_int64, ctypes.c_uint32, ctypes.c_double, ctypes.c_int
        lib.srt3d_ref_sketch.argtypes = [P, P, i64, u32, u32, i32, P]
        lib.srt3d_ref_phase_index.argtypes = [P, i64, u32, u32, P]
        lib.srt3d_ref_expected_sketch.argtypes = [P, P, i64, u32, f64, u32, u32, P]
        lib.srt3d_ref_sketch_grad.argtypes = [P, P, P, i64, u32, f64, u32, u32, P, P, P]
        lib.srt3d_ref_descent_update.argtypes = [P, P, P, P, i64, u32, f64, u32, u32, f64]
        lib.srt3d_ref_backproject.argtypes = [P, i64, f64, u32, u32, u32, P]
        lib.srt3d_ref_init_depths.argtypes = [P, i64, f64, u32, u32, u32, u32, u32, P, P, P, P]
        lib.srt3d_ref_init_k1.argtypes = [P, i64, f64, u32, u32, P, P]
        lib.srt3d_ref_sketch_merge.argtypes = [P, P, P, P, i64, u32, P, P]
        lib.srt3d_ref_bucket_events.argtypes = [P, P, ctypes.c_uint64, i64, P, P, P]
        for f in ("srt3d_ref_sketch", "srt3d_ref_phase_index", "srt3d_ref_expected_sketch",
                  "srt3d_ref_sketch_grad", "srt3d_ref_descent_update", "srt3d_ref_backproject",
                  "srt3d_ref_init_depths", "srt3d_ref_init_k1", "srt3d_ref_sketch_merge",
                  "srt3d_ref_bucket_events"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _check(rc: int, name: str):
    if rc != 0:
        raise ValueError(f"{name} returned {rc}")


def sketch(bins, offsets, T: int, m: int, mode: str = "exact") -> np.ndarray:
    """Eq. (3): complex128 z of shape (npix, m).

    mode="exact": integer reduction r=(j*x) mod T + libm table;
    mode="literal": libm cos/sin of the unreduced 2*pi*j*x/T."""
    bins = np.ascontiguousarray(bins, dtype=np.uint16)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint32)
    npix = offsets.size - 1
    z = np.zeros((max(npix, 0), m, 2), dtype=np.float64)
    rc = _load().srt3d_ref_sketch(_ptr(bins), _ptr(offsets), npix, T, m, 0 if mode == "exact" else 1, _ptr(z))
    _check(rc, "srt3d_ref_sketch")
    return z[..., 0] + 1j * z[..., 1]


def phase_index(bins, T: int, m: int) -> np.ndarray:
    """r[p, j-1] = (j * x_p) mod T (uint32), shape (n, m)."""
    bins = np.ascontiguousarray(bins, dtype=np.uint16)
    r = np.zeros((bins.size, m), dtype=np.uint32)
    _check(_load().srt3d_ref_phase_index(_ptr(bins), bins.size, T, m, _ptr(r)), "srt3d_ref_phase_index")
    return r


def expected_sketch(t, alpha, sigma: float, T: int, m: int) -> np.ndarray:
    """Eq. (4) with Gaussian hhat: complex128 (npix, m).

    t, alpha: (npix, K) — fp32 inputs are widened exactly to double."""
    t = np.ascontiguousarray(t, dtype=np.float64)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    npix, K = t.shape
    z = np.zeros((npix, m, 2), dtype=np.float64)
    rc = _load().srt3d_ref_expected_sketch(_ptr(t), _ptr(alpha), npix, K, float(sigma), T, m, _ptr(z))
    _check(rc, "srt3d_ref_expected_sketch")
    return z[..., 0] + 1j * z[..., 1]


def sketch_grad(z, t, alpha, sigma: float, T: int, m: int):
    """Eq. (6)/(8) data term (W=I, no n weight) and its gradient, in fp64.

    z: complex (npix, m); t, alpha: (npix, K).  Inputs are used exactly as
    given (complex64/float32 arrays are widened exactly), so for parity pass
    the very values the GPU consumed.  Returns (grad_t, grad_alpha, loss)."""
    z = np.asarray(z)
    zd = np.ascontiguousarray(np.stack([z.real, z.imag], axis=-1), dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    npix, K = t.shape
    gt = np.zeros((npix, K), dtype=np.float64)
    ga = np.zeros((npix, K), dtype=np.float64)
    loss = np.zeros(npix, dtype=np.float64)
    rc = _load().srt3d_ref_sketch_grad(_ptr(zd), _ptr(t), _ptr(alpha), npix, K, float(sigma), T, m,
                                       _ptr(gt), _ptr(ga), _ptr(loss))
    _check(rc, "srt3d_ref_sketch_grad")
    return gt, ga, loss


def descent_update(t, alpha, grad_t, grad_alpha, sigma: float, T: int, m: int, eta: float = 0.5):
    """Harness update (reading A13), fp64; returns new (t, alpha)."""
    t = np.array(t, dtype=np.float64, order="C", copy=True)
    alpha = np.array(alpha, dtype=np.float64, order="C", copy=True)
    gt = np.ascontiguousarray(grad_t, dtype=np.float64)
    ga = np.ascontiguousarray(grad_alpha, dtype=np.float64)
    npix, K = t.shape
    rc = _load().srt3d_ref_descent_update(_ptr(t), _ptr(alpha), _ptr(gt), _ptr(ga), npix, K,
                                          float(sigma), T, m, float(eta))
    _check(rc, "srt3d_ref_descent_update")
    return t, alpha


def _zd(z):
    z = np.asarray(z)
    return np.ascontiguousarray(np.stack([z.real, z.imag], axis=-1), dtype=np.float64)


def backproject(z, sigma: float, T: int, N: int) -> np.ndarray:
    """NEXT-3 (A18): g (npix, N), g[i, n] = Re sum_l z_l hhat_l e^{-i omega_l n T / N}."""
    zd = _zd(z)
    npix, m = zd.shape[0], zd.shape[1]
    g = np.zeros((npix, N), dtype=np.float64)
    _check(_load().srt3d_ref_backproject(_ptr(zd), npix, float(sigma), T, m, N, _ptr(g)), "srt3d_ref_backproject")
    return g


def init_depths(g, sigma: float, T: int, m: int, K: int, min_sep: int):
    """NEXT-3 (A19): greedy picks from a backprojection g (npix, N).
    Returns (t (npix, K), g_at_picks (npix, K), alpha (npix, K), count (npix,))."""
    g = np.ascontiguousarray(g, dtype=np.float64)
    npix, N = g.shape
    t = np.zeros((npix, K))
    gv = np.zeros((npix, K))
    a = np.zeros((npix, K))
    c = np.zeros(npix, dtype=np.int32)
    rc = _load().srt3d_ref_init_depths(_ptr(g), npix, float(sigma), T, m, N, K, int(min_sep), _ptr(t), _ptr(gv),
                                       _ptr(a), _ptr(c))
    _check(rc, "srt3d_ref_init_depths")
    return t, gv, a, c


def init_k1(z, sigma: float, T: int):
    """NEXT-3 (A20): K = 1 closed-form depth from arg(z_1) and least-squares alpha.
    Returns (t (npix,), alpha (npix,))."""
    zd = _zd(z)
    npix, m = zd.shape[0], zd.shape[1]
    t = np.zeros(npix)
    a = np.zeros(npix)
    _check(_load().srt3d_ref_init_k1(_ptr(zd), npix, float(sigma), T, m, _ptr(t), _ptr(a)), "srt3d_ref_init_k1")
    return t, a


def sketch_merge(za, na, zb, nb):
    """NEXT-4: count-weighted mean of two sketch frames; returns (z complex128 (npix, m), n uint64)."""
    a, b = _zd(za), _zd(zb)
    npix, m = a.shape[0], a.shape[1]
    na = np.ascontiguousarray(na, dtype=np.uint32)
    nb = np.ascontiguousarray(nb, dtype=np.uint32)
    z = np.zeros((npix, m, 2))
    n = np.zeros(npix, dtype=np.uint64)
    _check(_load().srt3d_ref_sketch_merge(_ptr(a), _ptr(na), _ptr(b), _ptr(nb), npix, m, _ptr(z), _ptr(n)),
           "srt3d_ref_sketch_merge")
    return z[..., 0] + 1j * z[..., 1], n


def bucket_events(pix, bins, npix: int):
    """NEXT-4: stable counting sort of (pixel, bin) events -> (offsets uint32 (npix+1,), bins uint16, dropped)."""
    pix = np.ascontiguousarray(pix, dtype=np.uint32)
    bins = np.ascontiguousarray(bins, dtype=np.uint16)
    offs = np.zeros(npix + 1, dtype=np.uint32)
    out = np.zeros(max(bins.size, 1), dtype=np.uint16)
    dropped = np.zeros(1, dtype=np.uint64)
    _check(_load().srt3d_ref_bucket_events(_ptr(pix), _ptr(bins), bins.size, npix, _ptr(offs), _ptr(out),
                                           _ptr(dropped)), "srt3d_ref_bucket_events")
    return offs, out[: int(offs[-1])], int(dropped[0])


def set_threads(n: int) -> None:
    """Set the OpenMP thread count used by the oracle (cpu_baseline 'cores')."""
    lib = ctypes.CDLL(None)
    try:
        _load()
        gomp = ctypes.CDLL("libgomp.so.1")
        gomp.omp_set_num_threads(ctypes.c_int(int(n)))
    except OSError:
        os.environ["OMP_NUM_THREADS"] = str(int(n))
    del lib


def max_threads() -> int:
    try:
        _load()
        gomp = ctypes.CDLL("libgomp.so.1")
        return int(gomp.omp_get_max_threads())
    except OSError:
        return 1
