"""Pixel sharding of a frame across ranks (one process per GPU).

Both kernels are independent per pixel, so a frame splits
into contiguous pixel blocks with no data-path collective: each rank sketches
and fits its own block.  A rank's CSR slice is the photon range
[offsets[i0], offsets[i1]) with offsets rebased to 0 (the C ABI also accepts
an un-rebased slice: offsets[0] may be non-zero)."""
from __future__ import annotations

import numpy as np


def pixel_range(npix: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous block [i0, i1) of ``npix`` pixels for ``rank``."""
    base, rem = divmod(npix, world)
    i0 = rank * base + min(rank, rem)
    return i0, i0 + base + (1 if rank < rem else 0)


def shard_csr(bins: np.ndarray, offsets: np.ndarray, i0: int, i1: int):
    """Rebased CSR of pixels [i0, i1): (bins slice, uint32 offsets of length i1-i0+1)."""
    p0, p1 = int(offsets[i0]), int(offsets[i1])
    offs = (offsets[i0:i1 + 1].astype(np.int64) - p0).astype(np.uint32)
    return bins[p0:p1], offs


def gather_rows(parts, npix: int, world: int):
    """Reassemble per-rank results (in rank order) into the full-frame array."""
    out = np.concatenate(parts, axis=0)
    assert out.shape[0] == npix
    return out
