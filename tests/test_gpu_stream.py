"""NEXT-4 GPU <-> oracle parity: sketch merge and event bucketing
through the C ABI.

  * bucketing: offsets bit-exact; dropped-event count exact; frames of up to
    512 * 8192 pixels (the two-level path) are a STABLE sort by pixel, so the
    output equals the oracle's stable counting sort bit for bit and is
    reproducible run to run; larger frames (one-level atomic
    path) follow atomic arrival inside a pixel: each pixel's bin multiset is
    bit-exact.
  * events -> CSR -> srt3d_sketch: |delta| <= 1e-5 per component vs the oracle's
    sketch of its own (stable) CSR (Eq. (3) is order-invariant; fp32 rounding
    order differs).
  * merge: |delta| <= 2e-7 * (|z_a| + |z_b|) + 1e-12 per component (weights
    rounded once to fp32, one FMA + one product).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _events(npix, T, n_ev, seed, extra_bad=0):
    rng = np.random.default_rng(seed)
    w = rng.exponential(1.0, npix)
    w[rng.random(npix) < 0.1] = 0.0  # empty pixels
    p = rng.choice(npix, size=n_ev, p=w / w.sum()).astype(np.uint32)
    if extra_bad:
        p[rng.choice(n_ev, extra_bad, replace=False)] = npix + rng.integers(0, 7, extra_bad)
    b = rng.integers(0, T, n_ev).astype(np.uint16)
    return p, b


@pytest.mark.parametrize("npix,T,n_ev,bad", [(1000, 4096, 200000, 0), (262144, 8192, 1000000, 17),
                                             (5000, 1024, 0, 0), (1, 100, 5000, 3), (70000, 2500, 300000, 0),
                                             (513, 4096, 40000, 5), (4194304, 1024, 300000, 0),
                                             (5000000, 2048, 200000, 2), (9000000, 1024, 100000, 1)])
def test_bucket_events_parity(gpu, oracle_mod, npix, T, n_ev, bad):
    import torch

    p, b = _events(npix, T, n_ev, seed=npix + n_ev, extra_bad=bad)
    offs, out, dropped = gpu.srt3d_bucket_events(_dev(p), _dev(b), npix)
    torch.cuda.synchronize()
    oo, ob, od = oracle_mod.bucket_events(p, b, npix)
    offs = offs.cpu().numpy()
    assert np.array_equal(offs, oo) and int(dropped.item()) == od == bad
    out = out.cpu().numpy()[: int(oo[-1])]
    if npix <= 512 * 8192:  # two-level path: stable, bitwise the oracle's order
        assert np.array_equal(out, ob)
        offs2, out2, _ = gpu.srt3d_bucket_events(_dev(p), _dev(b), npix)
        torch.cuda.synchronize()
        assert np.array_equal(out2.cpu().numpy()[: int(oo[-1])], out)  # run to run
    else:  # per-pixel multisets: sort inside every segment (keys: pixel, then bin)
        seg = np.repeat(np.arange(npix), np.diff(oo.astype(np.int64)))
        assert np.array_equal(out[np.lexsort((out, seg))], ob[np.lexsort((ob, seg))])


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_bucket_events_alignment_and_tails(gpu, oracle_mod, offset):
    """Pass A reads the pixel ids with 16-byte loads when the buffer is 16-byte aligned and
    element by element otherwise: a pixel buffer starting 0-3 elements into an
    allocation, an event count with a ragged last chunk (n mod 4 != 0), dropped events."""
    import torch

    npix, T, n_ev = 70001, 2048, 3 * 32768 + 4097
    p, b = _events(npix, T, n_ev, seed=offset + 11, extra_bad=3)
    dp = torch.zeros(p.size + 4, dtype=torch.int32, device="cuda")
    db = torch.zeros(b.size + 4, dtype=torch.int16, device="cuda")
    dp[offset: offset + p.size] = _dev(p.view(np.int32))
    db[offset: offset + b.size] = _dev(b.view(np.int16))
    pv = dp[offset: offset + p.size].view(torch.uint32)
    bv = db[offset: offset + b.size].view(torch.uint16)
    offs, out, dropped = gpu.srt3d_bucket_events(pv, bv, npix)
    torch.cuda.synchronize()
    oo, ob, od = oracle_mod.bucket_events(p, b, npix)
    assert np.array_equal(offs.cpu().numpy(), oo) and int(dropped.item()) == od == 3
    assert np.array_equal(out.cpu().numpy()[: int(oo[-1])], ob)


@pytest.mark.parametrize("T,m", [(8192, 32), (4613, 10), (1024, 4)])
def test_events_to_sketch(gpu, oracle_mod, T, m):
    import torch

    npix = 3000
    p, b = _events(npix, T, 600000, seed=T)
    offs, out, _ = gpu.srt3d_bucket_events(_dev(p), _dev(b), npix)
    z = gpu.srt3d_sketch(out, offs, T, m, total_photons=len(p))
    torch.cuda.synchronize()
    oo, ob, _ = oracle_mod.bucket_events(p, b, npix)
    zo = oracle_mod.sketch(ob, oo, T, m)
    zg = z.cpu().numpy()
    assert max(np.abs(zg.real - zo.real).max(), np.abs(zg.imag - zo.imag).max()) <= 1e-5


@pytest.mark.parametrize("m", [1, 10, 32, 64])
def test_sketch_merge_parity(gpu, oracle_mod, inputs_mod, m):
    """Random sketches and counts (incl. zero counts); out of place, then in place (z_out = z_a,
    n_out = n_a) — bitwise equal; merging two batch sketches equals the sketch of the union."""
    import torch

    rng = np.random.default_rng(m)
    npix = 5001
    za = (rng.normal(size=(npix, m)) + 1j * rng.normal(size=(npix, m))).astype(np.complex64)
    zb = (rng.normal(size=(npix, m)) + 1j * rng.normal(size=(npix, m))).astype(np.complex64)
    na = rng.integers(0, 3000, npix).astype(np.uint32)
    nb = rng.integers(0, 3000, npix).astype(np.uint32)
    na[:7] = 0
    nb[3:9] = 0
    zo, no = oracle_mod.sketch_merge(za, na, zb, nb)
    da, db, dna, dnb = _dev(za), _dev(zb), _dev(na), _dev(nb)
    z1, n1 = gpu.srt3d_sketch_merge(da, dna, db, dnb)
    torch.cuda.synchronize()
    z1h = z1.cpu().numpy()
    tol = 2e-7 * (np.abs(za) + np.abs(zb)) + 1e-12
    assert np.all(np.abs(z1h.real - zo.real) <= tol) and np.all(np.abs(z1h.imag - zo.imag) <= tol)
    assert np.array_equal(n1.cpu().numpy().astype(np.uint64), no)
    gpu.srt3d_sketch_merge(da, dna, db, dnb, z_out=da, n_out=dna)
    torch.cuda.synchronize()
    assert np.array_equal(da.cpu().numpy().view(np.uint64), z1h.view(np.uint64))
    assert np.array_equal(dna.cpu().numpy(), n1.cpu().numpy())
    # streaming: sketch of batch A merged with sketch of batch B == sketch of A u B
    T = 4096
    b1, o1 = inputs_mod.random_csr(npix=400, T=T, max_n=500, seed=1)
    b2, o2 = inputs_mod.random_csr(npix=400, T=T, max_n=500, seed=2)
    s1 = gpu.srt3d_sketch(_dev(b1), _dev(o1), T, m, total_photons=int(o1[-1]))
    s2 = gpu.srt3d_sketch(_dev(b2), _dev(o2), T, m, total_photons=int(o2[-1]))
    zm, nm = gpu.srt3d_sketch_merge(s1, _dev(np.diff(o1.astype(np.int64)).astype(np.uint32)), s2,
                                    _dev(np.diff(o2.astype(np.int64)).astype(np.uint32)))
    torch.cuda.synchronize()
    lists = [np.concatenate([b1[o1[i]:o1[i + 1]], b2[o2[i]:o2[i + 1]]]) for i in range(400)]
    ou = np.zeros(401, np.uint32)
    ou[1:] = np.cumsum([len(x) for x in lists])
    zu = oracle_mod.sketch(np.concatenate(lists).astype(np.uint16), ou, T, m)
    zmh = zm.cpu().numpy()
    assert max(np.abs(zmh.real - zu.real).max(), np.abs(zmh.imag - zu.imag).max()) <= 1e-5
    assert np.array_equal(nm.cpu().numpy(), np.diff(ou.astype(np.int64)).astype(np.uint32))


def test_stream_errors(gpu):
    import torch

    n = torch.zeros(4, dtype=torch.uint32, device="cuda")
    z65 = torch.zeros((4, 65), dtype=torch.complex64, device="cuda")
    with pytest.raises(gpu.Srt3dError):
        gpu.srt3d_sketch_merge(z65, n, z65, n)  # m > SRT3D_MAX_M
    assert gpu.srt3d_bucket_scratch_words(262144, 1000) >= 1000


@pytest.mark.parametrize("T,m", [(4096, 10), (8192, 32)])
def test_streaming_sketcher_equals_batch_sketch(gpu, oracle_mod, T, m):
    """PAPER.md:65 online acquisition: three event batches folded by StreamingSketcher
    (bucket -> sketch -> accumulate) equal the sketch of all kept events at once; counts exact;
    out-of-range pixels dropped and counted; srt3d_sketch_accumulate == srt3d_sketch_merge."""
    import torch

    from paper_2203_00952_b200.stream import StreamingSketcher

    npix = 2000
    batches = [_events(npix, T, n, seed=T + n, extra_bad=b) for n, b in ((100000, 0), (37000, 4), (120000, 0))]
    st = StreamingSketcher(npix, T, m, max_batch=120000)
    for p, b in batches:
        st.add(_dev(p), _dev(b))
    torch.cuda.synchronize()
    p_all = np.concatenate([p for p, _ in batches])
    b_all = np.concatenate([b for _, b in batches])
    oo, ob, od = oracle_mod.bucket_events(p_all, b_all, npix)
    zo = oracle_mod.sketch(ob, oo, T, m)
    zg = st.z.cpu().numpy()
    assert max(np.abs(zg.real - zo.real).max(), np.abs(zg.imag - zo.imag).max()) <= 1e-5
    assert np.array_equal(st.n.cpu().numpy(), np.diff(oo.astype(np.int64)).astype(np.uint32))
    assert int(st.dropped_total.item()) == od == 4
    # accumulate == merge with explicit counts
    offs, out, _ = gpu.srt3d_bucket_events(_dev(batches[0][0]), _dev(batches[0][1]), npix)
    zb = gpu.srt3d_sketch(out, offs, T, m, total_photons=100000)
    za, na = st.z.clone(), st.n.clone()
    nb = torch.from_numpy(np.diff(offs.cpu().numpy().astype(np.int64)).astype(np.uint32)).cuda()
    zm, nm = gpu.srt3d_sketch_merge(za, na, zb, nb)
    gpu.srt3d_sketch_accumulate(za, na, zb, offs)
    torch.cuda.synchronize()
    assert np.array_equal(za.cpu().numpy().view(np.uint64), zm.cpu().numpy().view(np.uint64))
    assert np.array_equal(na.cpu().numpy(), nm.cpu().numpy())


def test_streaming_bitwise_reproducible(gpu):
    """the streamed sketch (bucket -> sketch -> accumulate over batches) is bitwise
    identical run to run — the bucketing is a stable sort, so every kernel sees the same order."""
    import torch

    from paper_2203_00952_b200.stream import StreamingSketcher

    T, m, npix = 8192, 32, 262144
    batches = [_events(npix, T, n, seed=n) for n in (900000, 700000)]
    zs = []
    for _ in range(2):
        st = StreamingSketcher(npix, T, m, max_batch=900000)
        for p, b in batches:
            st.add(_dev(p), _dev(b))
        torch.cuda.synchronize()
        zs.append((st.z.cpu().numpy().copy(), st.n.cpu().numpy().copy()))
    assert np.array_equal(zs[0][0].view(np.uint64), zs[1][0].view(np.uint64))
    assert np.array_equal(zs[0][1], zs[1][1])
