"""paper_2203_00952_b200 — B200-native (sm_100a) hot path of sketched RT3D
(SRT3D, arxiv 2203.00952).

Thin Python binding of ``libsrt3d.so`` (C ABI in ``include/srt3d.h``):
argument marshalling only.  Every step of the path runs in the CUDA kernels
behind the ABI; there is no CPU or PyTorch fallback — if the library is
missing or a call fails, an exception is raised.

Functions take CUDA torch tensors (PyTorch provides device memory and
streams) and enqueue on the current torch stream unless ``stream`` is given:

  srt3d_sketch(bins, offsets, T, m, z=None)           Eq. (3)
  srt3d_expected_sketch(t, alpha, sigma, T, m)         Eq. (4)
  srt3d_sketch_grad(z, t, alpha, sigma, T, m)          Eq. (6)/(8) data term + gradient
  srt3d_descent_update(t, alpha, gt, ga, sigma, T, m, eta)   harness step (reading A13)
  srt3d_sketch_grad_step(z, t, alpha, sigma, T, m, eta)      fused grad + update
  srt3d_check_csr, srt3d_debug_phase_index            validation / test exports

``fit_frame`` / ``fit_frame_host`` run the whole hot path (sketch + N
gradient iterations) on device-resident or host (pinned) inputs.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsrt3d.so")
_lib = None

SRT3D_OK = 0
ERRORS = {-1: "SRT3D_EINVAL", -2: "SRT3D_ENULL", -3: "SRT3D_EUNSUPPORTED", -4: "SRT3D_ECUDA", -5: "SRT3D_EALIGN"}
PATH_AUTO, PATH_DIRECT, PATH_BINCOUNT, PATH_PAIRED, PATH_ROUTED, PATH_TENSOR = 0, 1, 2, 3, 4, 5
HINT_UNKNOWN = 0
EXPORTS = ("srt3d_version", "srt3d_last_error", "srt3d_sketch", "srt3d_sketch_ex", "srt3d_expected_sketch",
           "srt3d_sketch_grad",
           "srt3d_descent_update", "srt3d_sketch_grad_step", "srt3d_check_csr", "srt3d_debug_phase_index",
           "srt3d_sketch_plan", "srt3d_fit_pixelwise",
           "srt3d_backproject", "srt3d_init_depths", "srt3d_init_k1", "srt3d_sketch_merge",
           "srt3d_bucket_events", "srt3d_bucket_scratch_words", "srt3d_sketch_accumulate", "srt3d_debug_ffma_peak")


class Srt3dError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


def load_library(path: str | None = None):
    """Load libsrt3d.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA extension is required; there is no CPU fallback)")
    lib = ctypes.CDLL(p)
    P, i64, u32, u64, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_float
    lib.srt3d_version.argtypes = []
    lib.srt3d_version.restype = ctypes.c_int
    lib.srt3d_last_error.argtypes = []
    lib.srt3d_last_error.restype = ctypes.c_char_p
    lib.srt3d_sketch.argtypes = [P, P, i64, u32, u32, P, P]
    lib.srt3d_sketch_ex.argtypes = [P, P, i64, u32, u32, P, u64, ctypes.c_int, ctypes.c_int, P]
    lib.srt3d_expected_sketch.argtypes = [P, P, i64, u32, f32, u32, u32, P, P]
    lib.srt3d_sketch_grad.argtypes = [P, P, P, i64, u32, f32, u32, u32, P, P, P, P]
    lib.srt3d_descent_update.argtypes = [P, P, P, P, i64, u32, f32, u32, u32, f32, P]
    lib.srt3d_sketch_grad_step.argtypes = [P, P, P, i64, u32, f32, u32, u32, f32, P, P]
    lib.srt3d_check_csr.argtypes = [P, P, i64, u32, P, P]
    lib.srt3d_debug_phase_index.argtypes = [P, i64, u32, u32, P, P]
    lib.srt3d_sketch_plan.argtypes = [i64, u32, u32, u64, P]
    lib.srt3d_fit_pixelwise.argtypes = [P, P, P, i64, u32, f32, u32, u32, f32, u32, P, P]
    lib.srt3d_backproject.argtypes = [P, i64, f32, u32, u32, u32, P, P]
    lib.srt3d_init_depths.argtypes = [P, i64, f32, u32, u32, u32, u32, u32, P, P, P, P, P]
    lib.srt3d_init_k1.argtypes = [P, i64, f32, u32, u32, P, P, P]
    lib.srt3d_sketch_merge.argtypes = [P, P, P, P, i64, u32, P, P, P]
    lib.srt3d_bucket_events.argtypes = [P, P, u64, i64, P, P, P, P, P]
    lib.srt3d_sketch_accumulate.argtypes = [P, P, P, P, i64, u32, P]
    lib.srt3d_debug_ffma_peak.argtypes = [P]
    lib.srt3d_bucket_scratch_words.argtypes = [i64, u64]
    for f in EXPORTS[2:]:
        getattr(lib, f).restype = ctypes.c_int
    lib.srt3d_bucket_scratch_words.restype = u64  # size_t, not a status code
    if path is None:
        _lib = lib
    return lib


def _call(fn_name: str, *args):
    lib = load_library()
    rc = getattr(lib, fn_name)(*args)
    if rc != SRT3D_OK:
        raise Srt3dError(rc, lib.srt3d_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ValueError("all tensors must be contiguous CUDA tensors")


def _bins_ptr(bins, offsets):
    # an empty photon array has no storage; any valid device pointer will do
    # (no pixel owns a photon, so the kernels never dereference it)
    return _ptr(bins) if bins.numel() else _ptr(offsets)


def srt3d_sketch(bins: torch.Tensor, offsets: torch.Tensor, T: int, m: int, z: torch.Tensor | None = None,
                 total_photons: int | None = None, stream=None) -> torch.Tensor:
    """Eq. (3): complex64 (npix, m) sketch of a uint16/uint32 CSR frame on the GPU.

    Without ``total_photons`` this is the C ``srt3d_sketch`` (launch regime chosen on
    the device, no host read); with it, ``srt3d_sketch_ex`` with the hint (only the
    selected kernel is enqueued)."""
    npix = offsets.numel() - 1
    if z is None:
        z = torch.empty((max(npix, 0), m), dtype=torch.complex64, device=offsets.device)
    _need_cuda(bins, offsets, z)
    assert bins.dtype == torch.uint16 and offsets.dtype == torch.uint32 and z.dtype == torch.complex64
    if total_photons is None:
        _call("srt3d_sketch", _bins_ptr(bins, offsets), _ptr(offsets), npix, T, m, _ptr(z), _stream(stream))
    else:
        _call("srt3d_sketch_ex", _bins_ptr(bins, offsets), _ptr(offsets), npix, T, m, _ptr(z), int(total_photons),
              PATH_AUTO, 0, _stream(stream))
    return z


def srt3d_sketch_ex(bins: torch.Tensor, offsets: torch.Tensor, T: int, m: int, z: torch.Tensor | None = None,
                    total_photons: int | None = None, path: int = PATH_AUTO, lanes_per_pixel: int = 0,
                    stream=None) -> torch.Tensor:
    """Eq. (3) with the launch regime chosen explicitly (PATH_DIRECT with lanes 4..32, PATH_BINCOUNT, PATH_PAIRED);
    total_photons=None: HINT_UNKNOWN (regime picked on the device)."""
    npix = offsets.numel() - 1
    if z is None:
        z = torch.empty((max(npix, 0), m), dtype=torch.complex64, device=offsets.device)
    _need_cuda(bins, offsets, z)
    hint = int(total_photons) if total_photons is not None else HINT_UNKNOWN
    _call("srt3d_sketch_ex", _bins_ptr(bins, offsets), _ptr(offsets), npix, T, m, _ptr(z), hint, int(path),
          int(lanes_per_pixel), _stream(stream))
    return z


def srt3d_expected_sketch(t: torch.Tensor, alpha: torch.Tensor, sigma: float, T: int, m: int,
                          z: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Eq. (4) with Gaussian hhat: complex64 (npix, m)."""
    npix, K = t.shape
    if z is None:
        z = torch.empty((npix, m), dtype=torch.complex64, device=t.device)
    _need_cuda(t, alpha, z)
    _call("srt3d_expected_sketch", _ptr(t), _ptr(alpha), npix, K, float(sigma), T, m, _ptr(z), _stream(stream))
    return z


def srt3d_sketch_grad(z: torch.Tensor, t: torch.Tensor, alpha: torch.Tensor, sigma: float, T: int, m: int,
                      grad_t=None, grad_alpha=None, loss=None, want_loss: bool = True, stream=None):
    """Sketched loss ||z - Phi(theta)||^2 per pixel and its gradient (grad_t, grad_alpha, loss)."""
    npix, K = t.shape
    if grad_t is None:
        grad_t = torch.empty_like(t)
    if grad_alpha is None:
        grad_alpha = torch.empty_like(alpha)
    if loss is None and want_loss:
        loss = torch.empty(npix, dtype=torch.float32, device=t.device)
    _need_cuda(z, t, alpha, grad_t, grad_alpha, loss)
    _call("srt3d_sketch_grad", _ptr(z), _ptr(t), _ptr(alpha), npix, K, float(sigma), T, m, _ptr(grad_t),
          _ptr(grad_alpha), _ptr(loss), _stream(stream))
    return grad_t, grad_alpha, loss


def srt3d_descent_update(t, alpha, grad_t, grad_alpha, sigma: float, T: int, m: int, eta: float = 0.5, stream=None):
    """In-place harness update of (t, alpha) (reading A13)."""
    npix, K = t.shape
    _need_cuda(t, alpha, grad_t, grad_alpha)
    _call("srt3d_descent_update", _ptr(t), _ptr(alpha), _ptr(grad_t), _ptr(grad_alpha), npix, K, float(sigma), T, m,
          float(eta), _stream(stream))
    return t, alpha


def srt3d_sketch_grad_step(z, t, alpha, sigma: float, T: int, m: int, eta: float = 0.5, loss=None, stream=None):
    """Fused gradient + in-place update of (t, alpha); optional per-pixel loss."""
    npix, K = t.shape
    _need_cuda(z, t, alpha, loss)
    _call("srt3d_sketch_grad_step", _ptr(z), _ptr(t), _ptr(alpha), npix, K, float(sigma), T, m, float(eta),
          _ptr(loss), _stream(stream))
    return t, alpha


def srt3d_fit_pixelwise(z, t, alpha, sigma: float, T: int, m: int, iters: int, eta: float = 0.5, loss=None,
                        stream=None):
    """NEXT-2: `iters` fused data steps in one launch (t, alpha updated in place)."""
    npix, K = t.shape
    _need_cuda(z, t, alpha, loss)
    _call("srt3d_fit_pixelwise", _ptr(z), _ptr(t), _ptr(alpha), npix, K, float(sigma), T, m, float(eta), int(iters),
          _ptr(loss), _stream(stream))
    return t, alpha


def srt3d_backproject(z, sigma: float, T: int, N: int, g=None, stream=None):
    """NEXT-3: matched-filter backprojection on the circular grid t_n = n T / N: float32 (npix, N)."""
    npix, m = z.shape
    if g is None:
        g = torch.empty((npix, N), dtype=torch.float32, device=z.device)
    _need_cuda(z, g)
    _call("srt3d_backproject", _ptr(z), npix, float(sigma), T, m, N, _ptr(g), _stream(stream))
    return g


def srt3d_init_depths(z, sigma: float, T: int, N: int, K: int, min_sep: int, stream=None):
    """NEXT-3: up to K greedy backprojection peaks per pixel -> (t, g_at, alpha) float32 (npix, K),
    count int32 (npix,)."""
    npix, m = z.shape
    dev = z.device
    t = torch.empty((npix, K), dtype=torch.float32, device=dev)
    g = torch.empty_like(t)
    a = torch.empty_like(t)
    c = torch.empty(npix, dtype=torch.int32, device=dev)
    _need_cuda(z)
    _call("srt3d_init_depths", _ptr(z), npix, float(sigma), T, m, N, K, int(min_sep), _ptr(t), _ptr(g), _ptr(a),
          _ptr(c), _stream(stream))
    return t, g, a, c


def srt3d_init_k1(z, sigma: float, T: int, stream=None):
    """NEXT-3: K = 1 closed-form depth (phase of z_1) and least-squares alpha: float32 (npix, 1) each."""
    npix, m = z.shape
    t = torch.empty((npix, 1), dtype=torch.float32, device=z.device)
    a = torch.empty_like(t)
    _need_cuda(z)
    _call("srt3d_init_k1", _ptr(z), npix, float(sigma), T, m, _ptr(t), _ptr(a), _stream(stream))
    return t, a


def srt3d_sketch_merge(za, na, zb, nb, z_out=None, n_out=None, stream=None):
    """NEXT-4: count-weighted mean of two sketch frames (in place when z_out is za / n_out is na)."""
    npix, m = za.shape
    z_out = torch.empty_like(za) if z_out is None else z_out
    n_out = torch.empty_like(na) if n_out is None else n_out
    _need_cuda(za, na, zb, nb, z_out, n_out)
    _call("srt3d_sketch_merge", _ptr(za), _ptr(na), _ptr(zb), _ptr(nb), npix, m, _ptr(z_out), _ptr(n_out),
          _stream(stream))
    return z_out, n_out


def srt3d_sketch_accumulate(z, n, zb, offsets_b, stream=None):
    """NEXT-4: fold a batch sketch z_b (counts from its CSR offsets) into the running (z, n), in place."""
    npix, m = z.shape
    _need_cuda(z, n, zb, offsets_b)
    _call("srt3d_sketch_accumulate", _ptr(z), _ptr(n), _ptr(zb), _ptr(offsets_b), npix, m, _stream(stream))
    return z, n


def srt3d_debug_ffma_peak() -> float:
    """Measured FP32 FMA throughput of the current device now (TFLOP/s)."""
    v = ctypes.c_double(0.0)
    _call("srt3d_debug_ffma_peak", ctypes.byref(v))
    return float(v.value)


def srt3d_bucket_scratch_words(npix: int, nevents: int) -> int:
    """uint32 words of device workspace srt3d_bucket_events needs."""
    return int(load_library().srt3d_bucket_scratch_words(int(npix), int(nevents)))


def srt3d_bucket_events(pix, bins, npix: int, offsets=None, out=None, scratch=None, dropped=None, stream=None):
    """NEXT-4: unsorted (pixel uint32, bin uint16) events -> CSR (offsets uint32, bins uint16, dropped).
    Output / workspace tensors may be passed in (reused across batches)."""
    dev = pix.device
    nev = pix.numel()
    offsets = torch.empty(npix + 1, dtype=torch.uint32, device=dev) if offsets is None else offsets
    out = torch.empty(max(nev, 1), dtype=torch.uint16, device=dev) if out is None else out
    if scratch is None:
        scratch = torch.empty(max(1, srt3d_bucket_scratch_words(npix, nev)), dtype=torch.uint32, device=dev)
    dropped = torch.empty(1, dtype=torch.uint32, device=dev) if dropped is None else dropped
    if out.numel() < nev or scratch.numel() < srt3d_bucket_scratch_words(npix, nev) or offsets.numel() != npix + 1:
        raise ValueError("bucket_events: output / scratch tensors too small")
    _need_cuda(pix, bins)
    _call("srt3d_bucket_events", _ptr(pix), _ptr(bins), nev, int(npix), _ptr(offsets), _ptr(out), _ptr(scratch),
          _ptr(dropped), _stream(stream))
    return offsets, out, dropped


def srt3d_check_csr(bins, offsets, T: int, stream=None) -> int:
    npix = offsets.numel() - 1
    bad = torch.zeros(1, dtype=torch.int32, device=offsets.device)
    _need_cuda(bins, offsets)
    _call("srt3d_check_csr", _ptr(bins), _ptr(offsets), npix, T, _ptr(bad), _stream(stream))
    return int(bad.item())


def srt3d_debug_phase_index(bins, T: int, m: int, stream=None) -> torch.Tensor:
    n = bins.numel()
    r = torch.empty((n, m), dtype=torch.uint32, device=bins.device)
    _need_cuda(bins, r)
    _call("srt3d_debug_phase_index", _ptr(bins), n, T, m, _ptr(r), _stream(stream))
    return r


def fit_frame(bins, offsets, t0, alpha0, sigma: float, T: int, m: int, iters: int, eta: float = 0.5,
              total_photons: int | None = None, fused: bool = False, z=None, t=None, alpha=None, gt=None, ga=None,
              stream=None):
    """The whole hot path on device-resident inputs: sketch the frame (Eq. 3),
    then ``iters`` sketched-gradient iterations (Eq. 6/8 data step) from
    (t0, alpha0).  Returns (z, t, alpha)."""
    z = srt3d_sketch(bins, offsets, T, m, z=z, total_photons=total_photons, stream=stream)
    if t is None:
        t = t0.clone()
        alpha = alpha0.clone()
    else:
        t.copy_(t0)
        alpha.copy_(alpha0)
    if not fused:
        if gt is None:
            gt = torch.empty_like(t)
            ga = torch.empty_like(alpha)
    for _ in range(iters):
        if fused:
            srt3d_sketch_grad_step(z, t, alpha, sigma, T, m, eta, stream=stream)
        else:
            srt3d_sketch_grad(z, t, alpha, sigma, T, m, grad_t=gt, grad_alpha=ga, want_loss=False, stream=stream)
            srt3d_descent_update(t, alpha, gt, ga, sigma, T, m, eta, stream=stream)
    return z, t, alpha


def srt3d_sketch_plan(npix: int, T: int, m: int, total_photons: int):
    """(path, lanes_per_pixel) that srt3d_sketch uses for this frame shape (host-only query)."""
    lanes = ctypes.c_int(0)
    lib = load_library()
    rc = lib.srt3d_sketch_plan(int(npix), int(T), int(m), int(total_photons), ctypes.byref(lanes))
    if rc < 0:
        raise Srt3dError(rc, lib.srt3d_last_error().decode())
    return rc, lanes.value


def version() -> int:
    return int(load_library().srt3d_version())
