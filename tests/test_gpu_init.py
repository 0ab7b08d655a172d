"""NEXT-3 GPU <-> oracle parity: backprojection, greedy initial
depths and the K = 1 closed form, through the C ABI, on the same fp32 sketches.

Tolerances (readings A18-A20):
  * g: |delta| <= 1e-5 * S_i, S_i = sum_l hhat_l |z_il| (the triangle bound of g);
    Horner in fp32 over m <= 64 terms errs by <= 2 m eps S_i = 7.6e-6 S_i.
  * picks (integers decided by fp comparisons): identical where the oracle's
    decision is not a near-tie (margin > 2e-5 S_i); otherwise the GPU pick must be
    a valid choice within that margin.
  * init_k1: t within 0.5 fp32 ulp of T (both sides take fp64 atan2 of the same
    z_1; the GPU rounds t to fp32), circularly; alpha within 1e-4 * S_alpha,
    S_alpha = sum_l hhat_l |z_l| / sum_l hhat_l^2.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _hh(sigma, T, m):
    w = 2 * np.pi * np.arange(1, m + 1) / T
    return np.exp(-(sigma**2) * w**2 / 2)


def _gpu_sketch(gpu, bins, offs, T, m):
    import torch

    z = gpu.srt3d_sketch(_dev(bins), _dev(offs), T, m, total_photons=int(offs[-1]))
    torch.cuda.synchronize()
    return z


@pytest.mark.parametrize("T,m,N,sigma", [(1024, 4, 1024, 2.0), (4613, 10, 300, 5.0), (2500, 20, 129, 3.0),
                                         (8192, 32, 8192, 6.0), (8192, 64, 1000, 0.0), (100, 1, 7, 0.0),
                                         (17, 16, 1, 1.0), (4096, 10, 4096, 4.0),
                                         # tensor-core path (N % 32 == 0, N <= 512, m <= 32)
                                         (8192, 32, 512, 6.0), (4613, 10, 256, 5.0), (2500, 20, 32, 3.0),
                                         (1024, 1, 64, 2.0), (8192, 31, 480, 6.0), (4096, 17, 96, 0.0),
                                         # m > 32 at a tensor-core N: routed to the CUDA-core kernel
                                         (8192, 64, 512, 6.0)])
def test_backproject_parity(gpu, oracle_mod, inputs_mod, T, m, N, sigma):
    import torch

    bins, offs = inputs_mod.random_csr(npix=203, T=T, max_n=600, seed=T + m + N)
    z = _gpu_sketch(gpu, bins, offs, T, m)
    g = gpu.srt3d_backproject(z, sigma, T, N)
    torch.cuda.synchronize()
    zh = z.cpu().numpy()
    go = oracle_mod.backproject(zh, sigma, T, N)
    S = np.sum(_hh(sigma, T, m) * np.abs(zh), axis=1)[:, None]
    d = np.abs(g.cpu().numpy() - go)
    assert np.all(d <= 1e-5 * S + 1e-30), float((d / (S + 1e-30)).max())


def test_backproject_tc_many_tiles(gpu, oracle_mod, inputs_mod):
    """Tensor-core path over many 128-pixel tiles per persistent CTA (and a partial last tile):
    sampled rows against the oracle, plus init_depths picks on the same rows."""
    import torch

    T, m, N, sigma = 8192, 32, 512, 6.0
    npix = 148 * 128 * 2 + 77
    bins, offs = inputs_mod.random_csr(npix=npix, T=T, max_n=60, seed=5)
    z = _gpu_sketch(gpu, bins, offs, T, m)
    g = gpu.srt3d_backproject(z, sigma, T, N)
    tg, gg, ag, cg = gpu.srt3d_init_depths(z, sigma, T, N, 3, 50)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([[0, 127, 128, npix - 1], rng.choice(npix, 600, replace=False)]))
    zh = z.cpu().numpy()[idx]
    go = oracle_mod.backproject(zh, sigma, T, N)
    S = np.sum(_hh(sigma, T, m) * np.abs(zh), axis=1)[:, None]
    d = np.abs(g.cpu().numpy()[idx] - go)
    assert np.all(d <= 1e-5 * S + 1e-30), float((d / (S + 1e-30)).max())
    to, _, _, co = oracle_mod.init_depths(go, sigma, T, m, 3, 50)
    tgh, cgh = tg.cpu().numpy()[idx], cg.cpu().numpy()[idx]
    bad = _check_picks(tgh, cgh, 2e-5 * S[:, 0], to.astype(np.float32), co, lambda i: go[i], T, N, 50)
    assert bad <= len(idx) // 20, bad


def _check_picks(tg, cg, tol_g, to, co, go_row_fn, T, N, min_sep):
    """Exact match with the oracle's picks, or else the GPU's picks must be a greedy pick
    sequence (reading A19) of the oracle's g within tolerance tol (the GPU's g differs from
    the oracle's by <= tol): taken in descending g, each pick
      * is a candidate within tol (g > -tol, g > g_prev - tol, g >= g_next - tol),
      * keeps the minimum separation to every earlier pick,
      * is no smaller (beyond 2 tol) than any certain candidate (g > tol, g > g_prev + tol,
        g >= g_next + tol) still available after the earlier picks,
    and if fewer than K picks were made, no certain candidate remains available.  Counts
    that differ from the oracle's are accepted only under these rules.  Returns the number
    of pixels that did not match exactly (callers bound it)."""
    K = tg.shape[1]
    bad = 0
    for i in range(tg.shape[0]):
        if cg[i] == co[i] and np.array_equal(tg[i], to[i]):
            continue
        g = go_row_fn(i)
        # + the smallest normal fp32: g values below fp32's normal range (hhat ~ 1e-77 at T = 2,
        # sigma = 6) flush to zero on the GPU and cannot decide a pick
        tol = float(tol_g[i]) + float(np.finfo(np.float32).tiny)
        n_g = np.rint(tg[i, : cg[i]] * N / T).astype(np.int64) % N
        gp, gn = np.roll(g, 1), np.roll(g, -1)
        loose = (g > -tol) & (g > gp - tol) & (g >= gn - tol)
        certain = (g > tol) & (g > gp + tol) & (g >= gn + tol)
        grid = np.arange(N)

        def available(taken):
            ok = certain.copy()
            for q in taken:
                d = np.abs(grid - q)
                ok &= np.minimum(d, N - d) * T >= min_sep * N
            return ok

        taken = []
        for n in n_g[np.argsort(-g[n_g], kind="stable")]:
            assert loose[n], (i, int(n), "not a candidate")
            for q in taken:
                d = abs(int(n) - q)
                assert min(d, N - d) * T >= min_sep * N, (i, int(n), "separation")
            av = available(taken)
            if av.any():
                assert g[n] >= g[av].max() - 2 * tol, (i, int(n), "a clearly larger candidate was available")
            taken.append(int(n))
        if len(taken) < K:
            assert not available(taken).any(), (i, "stopped early although a certain candidate remained")
        bad += 1
    return bad


@pytest.mark.parametrize("T,m,N,K,min_sep,sigma", [(8192, 32, 512, 3, 50, 6.0), (2500, 20, 256, 2, 40, 3.0),
                                                   (1024, 4, 64, 1, 10, 2.0), (4613, 10, 4096, 8, 30, 5.0),
                                                   (100, 7, 3, 2, 1, 0.0)])
def test_init_depths_parity(gpu, oracle_mod, inputs_mod, T, m, N, K, min_sep, sigma):
    """Greedy picks on (a) noiseless multi-surface sketches (well separated: exact match required
    for every pixel) and (b) sketches of noisy ragged frames (near-ties allowed, see module doc)."""
    import torch

    rng = np.random.default_rng(T + K)
    npix = 150
    # (a) noiseless: K surfaces >= 4 * min_sep apart, alpha in [0.2, 1]
    Kt = min(K, 3)
    base = rng.uniform(0, T, npix)
    t = np.stack([(base + k * max(4 * min_sep, T // (Kt + 1))) % T for k in range(Kt)], axis=1).astype(np.float32)
    a = rng.uniform(0.2, 1.0, (npix, Kt)).astype(np.float32)
    z_a = gpu.srt3d_expected_sketch(_dev(t), _dev(a), sigma, T, m)
    # (b) noisy ragged frame
    bins, offs = inputs_mod.random_csr(npix=npix, T=T, max_n=400, seed=T + m)
    z_b = _gpu_sketch(gpu, bins, offs, T, m)
    for z, exact in ((z_a, True), (z_b, False)):
        tg, gg, ag, cg = gpu.srt3d_init_depths(z, sigma, T, N, K, min_sep)
        torch.cuda.synchronize()
        zh = z.cpu().numpy()
        gfull = oracle_mod.backproject(zh, sigma, T, N)
        to, go, ao, co = oracle_mod.init_depths(gfull, sigma, T, m, K, min_sep)
        tg, gg, ag, cg = (x.cpu().numpy() for x in (tg, gg, ag, cg))
        S = np.sum(_hh(sigma, T, m) * np.abs(zh), axis=1)
        tol = 2e-5 * S
        if exact and N >= 2 * m:
            match = (cg == co) & np.all(tg == to.astype(np.float32), axis=1)
            assert match.mean() >= 0.99, match.mean()
        bad = _check_picks(tg, cg, tol, to.astype(np.float32), co, lambda i: gfull[i], T, N, min_sep)
        assert bad <= max(2, npix // 20), bad
        same = (cg == co) & np.all(tg == to.astype(np.float32), axis=1)
        np.testing.assert_allclose(gg[same], go[same], atol=float(1e-5 * S.max()) + 1e-30)
        sh2 = np.sum(_hh(sigma, T, m) ** 2)
        assert np.all(np.abs(ag[same] - ao[same]) <= 1e-5 * S[same, None] / sh2 + 1e-6)
        assert np.all((ag >= 0) & (ag <= 1)) and np.all(cg <= K)


@pytest.mark.parametrize("cap", ["0", "2", "5"])
def test_init_depths_tc_list_overflow(gpu, oracle_mod, inputs_mod, monkeypatch, cap):
    """Tensor-core init_depths keeps each thread's candidates in a shared-memory list
    (DESIGN.md §5.5); a thread with more candidates than the list holds re-reads TMEM in
    its pick rounds and the next tile's MMAs wait for them.  Shrinking the list
    (SRT3D_INIT_LIST_CAP, read per launch) sends all (0) or some (2, 5) threads down that
    path over several tiles per CTA: the picks must be bitwise those of the default list,
    and match the oracle (near-ties as in _check_picks)."""
    import torch

    T, m, N, K, min_sep, sigma = 8192, 32, 512, 4, 40, 6.0
    npix = 148 * 128 + 300
    bins, offs = inputs_mod.random_csr(npix=npix, T=T, max_n=300, seed=77)
    z = _gpu_sketch(gpu, bins, offs, T, m)
    ref = [x.cpu().numpy() for x in gpu.srt3d_init_depths(z, sigma, T, N, K, min_sep)]
    monkeypatch.setenv("SRT3D_INIT_LIST_CAP", cap)
    out = [x.cpu().numpy() for x in gpu.srt3d_init_depths(z, sigma, T, N, K, min_sep)]
    torch.cuda.synchronize()
    for r, o in zip(ref, out):
        assert np.array_equal(r.view(np.uint32) if r.dtype == np.float32 else r,
                              o.view(np.uint32) if o.dtype == np.float32 else o)
    idx = np.random.default_rng(1).choice(npix, 300, replace=False)
    zh = z.cpu().numpy()[idx]
    gfull = oracle_mod.backproject(zh, sigma, T, N)
    to, go, ao, co = oracle_mod.init_depths(gfull, sigma, T, m, K, min_sep)
    S = np.sum(_hh(sigma, T, m) * np.abs(zh), axis=1)
    bad = _check_picks(out[0][idx], out[3][idx], 2e-5 * S, to.astype(np.float32), co, lambda i: gfull[i], T, N,
                       min_sep)
    assert bad <= 15, bad


def test_init_depths_edge_cases(gpu, oracle_mod):
    """Flat zero sketch -> no picks (A14 fill); K larger than the peaks; invalid args write nothing."""
    import torch

    T, m, N = 1024, 8, 256
    z = torch.zeros((5, m), dtype=torch.complex64, device="cuda")
    t, g, a, c = gpu.srt3d_init_depths(z, 1.0, T, N, 4, 10)
    torch.cuda.synchronize()
    assert np.all(c.cpu().numpy() == 0) and np.all(t.cpu().numpy() == T / 2) and np.all(a.cpu().numpy() == 0)
    for bad in (dict(N=2), dict(N=5000), dict(K=0), dict(K=9)):
        kw = dict(N=N, K=3)
        kw.update(bad)
        with pytest.raises(gpu.Srt3dError):
            gpu.srt3d_init_depths(z, 1.0, T, kw["N"], kw["K"], 10)
    with pytest.raises(gpu.Srt3dError):
        gpu.srt3d_backproject(z, 1.0, T, 9000)


@pytest.mark.parametrize("m", [16, 32, 48, 64])
def test_init_k1_tma_equals_cp_async(gpu, oracle_mod, inputs_mod, monkeypatch, m):
    """init_k1 stages z by TMA when m % 16 == 0; SRT3D_INIT_K1_CPASYNC=1
    forces the cp.async kernel.  Both must give bitwise the same t and alpha (same arithmetic)
    on a ragged frame with all-zero rows (the z_1 = 0 branch), and match the oracle."""
    import torch

    T, sigma, npix = 8192, 6.0, 148 * 128 + 45
    bins, offs = inputs_mod.random_csr(npix=npix, T=T, max_n=200, seed=m)
    z = _gpu_sketch(gpu, bins, offs, T, m)
    z[::97] = 0.0
    tg, ag = (x.cpu().numpy() for x in gpu.srt3d_init_k1(z, sigma, T))
    monkeypatch.setenv("SRT3D_INIT_K1_CPASYNC", "1")
    tc, ac = (x.cpu().numpy() for x in gpu.srt3d_init_k1(z, sigma, T))
    torch.cuda.synchronize()
    assert np.array_equal(tg.view(np.uint32), tc.view(np.uint32))
    assert np.array_equal(ag.view(np.uint32), ac.view(np.uint32))
    idx = np.random.default_rng(m).choice(npix, 400, replace=False)
    zh = z.cpu().numpy()[idx]
    to, ao = oracle_mod.init_k1(zh, sigma, T)
    d = np.abs(tg[idx, 0].astype(np.float64) - to)
    assert np.all(np.minimum(d, T - d) <= 0.5 * np.spacing(np.float32(T)) + 1e-9)
    h = _hh(sigma, T, m)
    Sa = np.sum(h * np.abs(zh), axis=1) / np.sum(h**2)
    assert np.all(np.abs(ag[idx, 0] - ao) <= 1e-4 * Sa + 1e-7)


@pytest.mark.parametrize("T,m,sigma", [(4613, 10, 5.0), (8192, 32, 6.0), (1024, 4, 2.0), (2500, 64, 0.0)])
def test_init_k1_parity(gpu, oracle_mod, inputs_mod, T, m, sigma):
    import torch

    rng = np.random.default_rng(T)
    npix = 500
    t = rng.uniform(0, T, (npix, 1)).astype(np.float32)
    t[:4, 0] = [0.0, T - 0.001, T / 2, 1e-3]
    a = rng.uniform(0.05, 1, (npix, 1)).astype(np.float32)
    z_a = gpu.srt3d_expected_sketch(_dev(t), _dev(a), sigma, T, m)
    bins, offs = inputs_mod.random_csr(npix=npix, T=T, max_n=300, seed=T + 1)
    z_b = _gpu_sketch(gpu, bins, offs, T, m)
    for z in (z_a, z_b):
        tg, ag = gpu.srt3d_init_k1(z, sigma, T)
        torch.cuda.synchronize()
        zh = z.cpu().numpy()
        to, ao = oracle_mod.init_k1(zh, sigma, T)
        tg, ag = tg.cpu().numpy()[:, 0], ag.cpu().numpy()[:, 0]
        d = np.abs(tg.astype(np.float64) - to)
        d = np.minimum(d, T - d)
        ulp = np.spacing(np.float32(T))
        assert np.all(d <= 0.5 * ulp + 1e-9), float(d.max())
        assert np.all((tg >= 0) & (tg < T))
        h = _hh(sigma, T, m)
        Sa = np.sum(h * np.abs(zh), axis=1) / np.sum(h**2)
        assert np.all(np.abs(ag - ao) <= 1e-4 * Sa + 1e-7), float(np.abs(ag - ao).max())
    # noiseless truth is recovered (z_a): t within 0.01 bins, alpha within 1e-4
    tg, ag = gpu.srt3d_init_k1(z_a, sigma, T)
    d = np.abs(tg.cpu().numpy() - t)
    assert np.all(np.minimum(d, T - d) < 0.01)
    np.testing.assert_allclose(ag.cpu().numpy(), a, atol=1e-4)
