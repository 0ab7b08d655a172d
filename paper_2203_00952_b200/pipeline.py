"""FramePipeline — the whole SRT3D hot path for one frame shape, replayed as
CUDA graphs.

One step = srt3d_sketch over the frame (Eq. 3) followed by ``iters``
sketched-gradient iterations (Eq. 6/8 data term + the A13 update) from
theta0.  Device buffers are allocated once (PyTorch owns them); the step is
captured as two CUDA graphs (sketch | theta reset + iterations) so a step
costs two graph launches instead of 1 + iters kernel launches from Python.

  run_device()            inputs already resident in HBM
  run_host(bins, offsets, t0, alpha0, t_out, alpha_out)
                          end to end from pinned host buffers: H2D copies of
                          the frame and theta0, the step, D2H of the fitted
                          theta — all stream-ordered on one stream.
"""
from __future__ import annotations

import torch

from . import srt3d_descent_update, srt3d_sketch, srt3d_sketch_grad, srt3d_sketch_grad_step


class FramePipeline:
    def __init__(self, n_photons: int, npix: int, K: int, T: int, m: int, sigma: float, iters: int,
                 eta: float = 0.5, fused: bool = True, use_graphs: bool = True, device=None):
        self.device = torch.device(device or "cuda")
        self.n_photons, self.npix, self.K, self.T, self.m = int(n_photons), int(npix), int(K), int(T), int(m)
        self.sigma, self.iters, self.eta, self.fused = float(sigma), int(iters), float(eta), bool(fused)
        d = self.device
        self.bins = torch.empty(max(self.n_photons, 1), dtype=torch.uint16, device=d)
        self.offsets = torch.empty(self.npix + 1, dtype=torch.uint32, device=d)
        self.t0 = torch.empty((self.npix, K), dtype=torch.float32, device=d)
        self.a0 = torch.empty((self.npix, K), dtype=torch.float32, device=d)
        self.z = torch.empty((self.npix, m), dtype=torch.complex64, device=d)
        self.t = torch.empty_like(self.t0)
        self.a = torch.empty_like(self.a0)
        self.gt = torch.empty_like(self.t0)
        self.ga = torch.empty_like(self.a0)
        self.stream = torch.cuda.Stream(device=d)
        self.use_graphs = use_graphs
        self.g_sketch = None
        self.g_iter = None

    # kernels launched per step (for the bench's gpu_launches claim)
    @property
    def launches_per_step(self) -> int:
        passes = (self.m + 31) // 32
        return passes + self.iters * (1 if self.fused else 2)

    def load_device(self, bins, offsets, t0, a0):
        with torch.cuda.stream(self.stream):
            self.bins[: bins.numel()].copy_(bins, non_blocking=True)
            self.offsets.copy_(offsets, non_blocking=True)
            self.t0.copy_(t0, non_blocking=True)
            self.a0.copy_(a0, non_blocking=True)
        self.stream.synchronize()

    def _sketch(self):
        srt3d_sketch(self.bins, self.offsets, self.T, self.m, z=self.z, total_photons=self.n_photons)

    def _iterate(self):
        self.t.copy_(self.t0)
        self.a.copy_(self.a0)
        for _ in range(self.iters):
            if self.fused:
                srt3d_sketch_grad_step(self.z, self.t, self.a, self.sigma, self.T, self.m, self.eta)
            else:
                srt3d_sketch_grad(self.z, self.t, self.a, self.sigma, self.T, self.m, grad_t=self.gt,
                                  grad_alpha=self.ga, want_loss=False)
                srt3d_descent_update(self.t, self.a, self.gt, self.ga, self.sigma, self.T, self.m, self.eta)

    def capture(self):
        """Run the step once eagerly (warms host-side caches), then capture it."""
        with torch.cuda.stream(self.stream):
            self._sketch()
            self._iterate()
        self.stream.synchronize()
        if not self.use_graphs:
            return
        self.g_sketch = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_sketch, stream=self.stream, capture_error_mode="thread_local"):
            self._sketch()
        self.g_iter = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.g_iter, stream=self.stream, capture_error_mode="thread_local"):
            self._iterate()
        self.stream.synchronize()

    def sketch_phase(self):
        """Enqueue the sketch on self.stream (graph replay or direct launch)."""
        with torch.cuda.stream(self.stream):
            if self.g_sketch is not None:
                self.g_sketch.replay()
            else:
                self._sketch()

    def iterate_phase(self):
        with torch.cuda.stream(self.stream):
            if self.g_iter is not None:
                self.g_iter.replay()
            else:
                self._iterate()

    def run_device(self):
        self.sketch_phase()
        self.iterate_phase()

    def run_host(self, bins_h, offsets_h, t0_h, a0_h, t_out_h, a_out_h):
        """End-to-end step from (pinned) host buffers; results land in t_out_h / a_out_h."""
        with torch.cuda.stream(self.stream):
            self.bins[: bins_h.numel()].copy_(bins_h, non_blocking=True)
            self.offsets.copy_(offsets_h, non_blocking=True)
            self.t0.copy_(t0_h, non_blocking=True)
            self.a0.copy_(a0_h, non_blocking=True)
        self.run_device()
        with torch.cuda.stream(self.stream):
            t_out_h.copy_(self.t, non_blocking=True)
            a_out_h.copy_(self.a, non_blocking=True)

    def h2d_bytes(self) -> int:
        return 2 * self.n_photons + 4 * (self.npix + 1) + 2 * 4 * self.npix * self.K

    def d2h_bytes(self) -> int:
        return 2 * 4 * self.npix * self.K
