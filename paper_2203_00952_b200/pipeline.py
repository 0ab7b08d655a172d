"""FramePipeline — the whole SRT3D hot path for one frame shape, replayed as
CUDA graphs.

One step = srt3d_sketch over the frame (Eq. 3) followed by ``iters``
sketched-gradient iterations (Eq. 6/8 data term + the A13 update) from
theta0.  Device buffers are allocated once (PyTorch owns them); the step is
captured as two CUDA graphs (sketch | theta reset + iterations) so a step
costs two graph launches instead of 1 + iters kernel launches from Python.

  run_device()            inputs already resident in HBM
  run_host(bins, offsets, t0, alpha0, t_out, alpha_out, chunks=1)
                          end to end from pinned host buffers: H2D copies of
                          the frame and theta0, the step, D2H of the fitted
                          theta.  With chunks > 1 the frame is split into
                          pixel blocks (pixels are independent): the copy
                          engine uploads block c+1 on its own stream while
                          the SMs sketch and iterate block c (one CUDA graph
                          per block), so PCIe and compute overlap;
                          chain=True lets consecutive frames stream back
                          to back (frame f+1's uploads overlap frame f's
                          last block).
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
        self.copy_stream = torch.cuda.Stream(device=d)
        self.use_graphs = use_graphs
        self.g_sketch = None
        self.g_iter = None
        self.chunk_bounds = None  # pixel boundaries of the pipelined host path
        self.g_chunks = []
        self.ev_in, self.ev_done = [], []

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

    def _sketch(self, i0: int = 0, i1: int | None = None):
        i1 = self.npix if i1 is None else i1
        hint = max(1, round(self.n_photons * (i1 - i0) / max(self.npix, 1)))  # selects the launch regime only
        srt3d_sketch(self.bins, self.offsets[i0:i1 + 1], self.T, self.m, z=self.z[i0:i1], total_photons=hint)

    def _iterate(self, i0: int = 0, i1: int | None = None, iters: int | None = None, reset: bool = True):
        i1 = self.npix if i1 is None else i1
        z, t, a, gt, ga = self.z[i0:i1], self.t[i0:i1], self.a[i0:i1], self.gt[i0:i1], self.ga[i0:i1]
        if reset:
            t.copy_(self.t0[i0:i1])
            a.copy_(self.a0[i0:i1])
        for _ in range(self.iters if iters is None else int(iters)):
            if self.fused:
                srt3d_sketch_grad_step(z, t, a, self.sigma, self.T, self.m, self.eta)
            else:
                srt3d_sketch_grad(z, t, a, self.sigma, self.T, self.m, grad_t=gt, grad_alpha=ga, want_loss=False)
                srt3d_descent_update(t, a, gt, ga, self.sigma, self.T, self.m, self.eta)

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

    def run_iterations(self, n: int, reset: bool = False):
        """Enqueue n more iterations of the step's own kernel on self.stream without
        graphs (reset=True first restores theta0): for per-iteration snapshots in tests."""
        with torch.cuda.stream(self.stream):
            self._iterate(iters=n, reset=reset)

    def capture_chunks(self, chunks: int):
        """Per-block graphs (sketch + theta reset + iterations) for run_host(chunks=...)."""
        chunks = max(1, min(int(chunks), self.npix))
        b = [(self.npix * c) // chunks for c in range(chunks + 1)]
        if self.chunk_bounds == b:
            return
        self.chunk_bounds = b
        self.g_chunks = []
        self.ev_in = [torch.cuda.Event() for _ in range(chunks)]
        self.ev_done = [torch.cuda.Event() for _ in range(chunks)]
        with torch.cuda.stream(self.stream):
            for c in range(chunks):  # eager run first (host-side caches, attributes)
                self._sketch(b[c], b[c + 1])
                self._iterate(b[c], b[c + 1])
        self.stream.synchronize()
        for c in range(chunks):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream, capture_error_mode="thread_local"):
                self._sketch(b[c], b[c + 1])
                self._iterate(b[c], b[c + 1])
            self.g_chunks.append(g)
        for ev in self.ev_done:
            ev.record(self.stream)
        self.stream.synchronize()

    def run_host(self, bins_h, offsets_h, t0_h, a0_h, t_out_h, a_out_h, chunks: int = 1, chain: bool = False):
        """End-to-end step from (pinned) host buffers; results land in t_out_h / a_out_h.
        chunks > 1: pipelined per pixel block (H2D of block c+1 overlaps compute of block c).
        chain=True (only directly after a chunked run_host with the same chunks, nothing else
        enqueued on this pipeline in between): the uploads of this frame do not wait for the
        previous frame's tail — block c is uploaded as soon as block c of the previous frame is
        done (ev_done[c]), so consecutive frames stream back to back over PCIe."""
        if chunks > 1:
            if chain and self.chunk_bounds is not None and len(self.chunk_bounds) - 1 == max(1, min(int(chunks), self.npix)):
                b = self.chunk_bounds
            else:
                self.capture_chunks(chunks)
                b = self.chunk_bounds
                self.copy_stream.wait_stream(self.stream)  # uploads start after work already queued (and timers)
            for c in range(len(b) - 1):
                i0, i1 = b[c], b[c + 1]
                p0, p1 = int(offsets_h[i0]), int(offsets_h[i1])
                with torch.cuda.stream(self.copy_stream):
                    self.copy_stream.wait_event(self.ev_done[c])  # block c of the previous step is done
                    if p1 > p0:
                        self.bins[p0:p1].copy_(bins_h[p0:p1], non_blocking=True)
                    self.offsets[i0:i1 + 1].copy_(offsets_h[i0:i1 + 1], non_blocking=True)
                    self.t0[i0:i1].copy_(t0_h[i0:i1], non_blocking=True)
                    self.a0[i0:i1].copy_(a0_h[i0:i1], non_blocking=True)
                    self.ev_in[c].record(self.copy_stream)
                with torch.cuda.stream(self.stream):
                    self.stream.wait_event(self.ev_in[c])
                    self.g_chunks[c].replay()
                    self.ev_done[c].record(self.stream)
                    t_out_h[i0:i1].copy_(self.t[i0:i1], non_blocking=True)
                    a_out_h[i0:i1].copy_(self.a[i0:i1], non_blocking=True)
            return
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
