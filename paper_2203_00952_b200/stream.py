"""StreamingSketcher — the acquisition-side use of the sketch ("it
can be updated in an online fashion with each incoming photon throughout the
duration of the acquisition time"; NEXT-4 of SURVEY §8(f)).

Photon events arrive in batches as unsorted (pixel index, bin) pairs.  Each
``add`` buckets the batch into a pixel-sorted CSR frame on the GPU
(srt3d_bucket_events), sketches it (srt3d_sketch, Eq. (3)) and folds it into
the running per-pixel sketch with its photon counts (srt3d_sketch_accumulate:
count-weighted mean).  Only z (npix x m complex) and the
counts persist between batches — no per-photon storage.
All buffers are allocated once; every step runs in libsrt3d.so.
"""
from __future__ import annotations

import torch

from . import srt3d_bucket_events, srt3d_bucket_scratch_words, srt3d_sketch, srt3d_sketch_accumulate


class StreamingSketcher:
    def __init__(self, npix: int, T: int, m: int, max_batch: int, device=None):
        self.npix, self.T, self.m, self.max_batch = int(npix), int(T), int(m), int(max_batch)
        d = torch.device(device or "cuda")
        self.z = torch.zeros((self.npix, self.m), dtype=torch.complex64, device=d)
        self.n = torch.zeros(self.npix, dtype=torch.uint32, device=d)
        self._zb = torch.empty_like(self.z)
        self._offs = torch.empty(self.npix + 1, dtype=torch.uint32, device=d)
        self._bins = torch.empty(max(self.max_batch, 1), dtype=torch.uint16, device=d)
        self._scratch = torch.empty(max(1, srt3d_bucket_scratch_words(self.npix, self.max_batch)), dtype=torch.uint32,
                                    device=d)
        self._dropped = torch.zeros(1, dtype=torch.uint32, device=d)
        self.dropped_total = torch.zeros(1, dtype=torch.int64, device=d)

    def add(self, pix: torch.Tensor, bins: torch.Tensor, stream=None):
        """Fold one batch of events (uint32 pixel ids, uint16 bins < T; same length <= max_batch)."""
        nev = pix.numel()
        if nev > self.max_batch or bins.numel() != nev:
            raise ValueError(f"batch of {nev} events (max {self.max_batch}) / bins of {bins.numel()}")
        srt3d_bucket_events(pix, bins, self.npix, offsets=self._offs, out=self._bins, scratch=self._scratch,
                            dropped=self._dropped, stream=stream)
        srt3d_sketch(self._bins, self._offs, self.T, self.m, z=self._zb, total_photons=max(nev, 1), stream=stream)
        srt3d_sketch_accumulate(self.z, self.n, self._zb, self._offs, stream=stream)
        self.dropped_total += self._dropped.to(torch.int64)
        return self

    def reset(self):
        self.z.zero_()
        self.n.zero_()
        self.dropped_total.zero_()
