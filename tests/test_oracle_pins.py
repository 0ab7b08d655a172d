"""Pins of the fp64 oracle against what the paper and the mathematics fix
(closed forms, special cases, brute force, finite differences, invariants).

Every check here is independent of the oracle's own code path: closed forms
are derived by hand from Eq. (3)/(4)/(6), brute-force sums run over the Eq. (1)
model distribution in numpy, and gradients are checked against central
finite differences of the loss.  Citations: PAPER.md line numbers (P:n),
SURVEY.md §8(c) pin ids (P1..P8, E1..E3, G1..G6, B1), DESIGN.md readings."""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _csr(lists):
    offs = np.zeros(len(lists) + 1, dtype=np.uint32)
    offs[1:] = np.cumsum([len(l) for l in lists])
    bins = np.concatenate([np.asarray(l, dtype=np.uint16) for l in lists]) if offs[-1] else np.zeros(0, np.uint16)
    return bins, offs


def _hhat(sigma, T, m):
    w = 2 * np.pi * np.arange(1, m + 1) / T
    return w, np.exp(-sigma**2 * w**2 / 2)


# ---------------------------------------------------------------- sketch, Eq. (3)
def test_P1_single_photon(oracle_mod):
    """P1: one photon at x gives z_j = exp(i 2 pi j x / T); T=100, x=25 -> (i, -1, -i, 1)."""
    b, o = _csr([[25]])
    z = oracle_mod.sketch(b, o, 100, 4)[0]
    np.testing.assert_allclose(z, [1j, -1, -1j, 1], atol=1e-15)
    for T, x, m in [(4613, 4612, 10), (8192, 1, 32), (65536, 65535, 64), (3, 2, 2)]:
        b, o = _csr([[x]])
        for mode in ("exact", "literal"):
            z = oracle_mod.sketch(b, o, T, m, mode=mode)[0]
            j = np.arange(1, m + 1)
            np.testing.assert_allclose(z, np.exp(2j * np.pi * ((j * x) % T) / T), atol=1e-12)


def test_P2_mean_of_terms_and_merge(oracle_mod):
    """P2: a sketch is the mean of per-photon terms; sketch(A u B) = (nA zA + nB zB)/(nA+nB),
    independent of photon order."""
    rng = np.random.default_rng(1)
    T, m = 4613, 10
    A = rng.integers(0, T, 37)
    B = rng.integers(0, T, 91)
    b, o = _csr([A, B, np.concatenate([B, A]), rng.permutation(np.concatenate([A, B]))])
    z = oracle_mod.sketch(b, o, T, m)
    merged = (len(A) * z[0] + len(B) * z[1]) / (len(A) + len(B))
    np.testing.assert_allclose(z[2], merged, atol=1e-14)
    np.testing.assert_allclose(z[3], merged, atol=1e-14)
    # mean of single-photon sketches
    singles = np.stack([oracle_mod.sketch(*_csr([[x]]), T, m)[0] for x in A])
    np.testing.assert_allclose(z[0], singles.mean(axis=0), atol=1e-14)


@pytest.mark.parametrize("T", [16, 100, 153, 1024])
def test_P3_uniform_background_is_blind(oracle_mod, T):
    """P3: one photon in every bin 0..T-1 sketches to 0 for all 1 <= j <= T-1
    (background blindness of omega_l = 2 pi l / T)."""
    m = min(T - 1, 64)
    b, o = _csr([np.arange(T)])
    z = oracle_mod.sketch(b, o, T, m)[0]
    assert np.abs(z).max() < 1e-13


def test_P4_small_closed_forms(oracle_mod):
    """P4: {0, T/2} -> z_j = (1 + (-1)^j)/2; {0, 25, 50} at T=100 -> z1 = i/3, z2 = 1/3."""
    T = 100
    b, o = _csr([[0, 50], [0, 25, 50]])
    z = oracle_mod.sketch(b, o, T, 6)
    j = np.arange(1, 7)
    np.testing.assert_allclose(z[0], (1 + (-1.0) ** j) / 2, atol=1e-15)
    np.testing.assert_allclose(z[1][:2], [1j / 3, 1 / 3], atol=1e-15)


def test_P5_shift_equivariance_and_conjugate_symmetry(oracle_mod):
    """P5: x -> (x+s) mod T multiplies z_j by exp(i 2 pi j s / T); z_{T-j} = conj(z_j)."""
    rng = np.random.default_rng(2)
    T, s = 64, 13
    x = rng.integers(0, T, 50)
    b, o = _csr([x, (x + s) % T])
    z = oracle_mod.sketch(b, o, T, T - 1)
    j = np.arange(1, T)
    np.testing.assert_allclose(z[1], z[0] * np.exp(2j * np.pi * j * s / T), atol=1e-13)
    np.testing.assert_allclose(z[0][::-1], np.conj(z[0]), atol=1e-13)  # z_{T-j} = conj z_j


def test_P6_literal_equals_exact_index(oracle_mod):
    """P6: literal libm of the unreduced argument equals the exact-index mode within 1e-12."""
    rng = np.random.default_rng(3)
    for T, m in [(1024, 4), (4613, 10), (65536, 64), (7, 6)]:
        lists = [rng.integers(0, T, rng.integers(0, 40)) for _ in range(20)]
        b, o = _csr(lists)
        np.testing.assert_allclose(oracle_mod.sketch(b, o, T, m, "literal"), oracle_mod.sketch(b, o, T, m, "exact"),
                                   atol=1e-12)


def test_P7_empty_pixels(oracle_mod):
    """P7: n = 0 gives z = 0 (reading A10), also between non-empty pixels."""
    b, o = _csr([[], [5], [], []])
    z = oracle_mod.sketch(b, o, 10, 3)
    assert np.all(z[[0, 2, 3]] == 0)
    np.testing.assert_allclose(z[1], np.exp(2j * np.pi * np.arange(1, 4) * 5 / 10), atol=1e-15)


def test_P8_clt_mean_sketch_matches_model(oracle_mod, inputs_mod):
    """P8: sketches of photons drawn from Eq. (1) average to Phi(theta) (Eq. 4/5) within
    a 5-sigma CLT bound.  Pins sketch + expected_sketch + the generator's law together."""
    T, sigma, m, npix, n = 1024, 2.0, 8, 400, 2000
    t = np.full((npix, 2), [300.3, 701.8], dtype=np.float32)
    w = np.tile([1.0, 0.6, 0.4], (npix, 1))  # background weight 1, surfaces 0.6 / 0.4
    bins, offs = inputs_mod.sample_photons(t, w, sigma, T, seed=7, fixed_n=n)
    z = oracle_mod.sketch(bins, offs, T, m).mean(axis=0)
    alpha = np.array([[0.3, 0.2]])
    phi = oracle_mod.expected_sketch(t[:1].astype(np.float64), alpha, sigma, T, m)[0]
    N = npix * n
    assert np.abs(z - phi).max() < 5.0 / np.sqrt(N)


# ------------------------------------------------------- expected sketch, Eq. (4)
def test_E1_closed_form_instance(oracle_mod):
    """E1: Phi_j = sum_k alpha_k exp(-sigma^2 w_j^2/2) exp(i w_j t_k) (Eq. 4); SURVEY §8(c) worked values."""
    with open(os.path.join(GOLDEN, "e1_expected_sketch.json")) as f:
        g = json.load(f)
    phi = oracle_mod.expected_sketch(np.array([g["t"]]), np.array([g["alpha"]]), g["sigma"], g["T"], g["m"])[0]
    for j, re, im in g["values"]:
        assert abs(phi[j - 1] - complex(re, im)) < 1e-15
    w, h = _hhat(g["sigma"], g["T"], g["m"])
    direct = (np.array(g["alpha"])[None, :] * h[:, None] * np.exp(1j * w[:, None] * np.array(g["t"])[None, :])).sum(1)
    np.testing.assert_allclose(phi, direct, atol=1e-16)


@pytest.mark.parametrize("T,sigma,K,j", [(1024, 2.0, 1, 4), (8192, 6.0, 3, 32), (4096, 4.0, 1, 10),
                                         (2500, 3.0, 2, 20), (153, 2.0, 2, 10)])
def test_E2_bruteforce_over_model_distribution(oracle_mod, T, sigma, K, j):
    """E2: Phi_j equals sum_{x=0}^{T-1} pi(x|theta) exp(i w_j x) for the Eq. (1) mixture
     with the wrapped discrete Gaussian IRF and a uniform background."""
    rng = np.random.default_rng(T + K)
    t = rng.uniform(0, T, K)
    alpha = rng.uniform(0.05, 0.3, K)
    alpha0 = 1 - alpha.sum()
    x = np.arange(T, dtype=np.float64)
    pi = np.full(T, alpha0 / T)
    for k in range(K):
        dens = sum(np.exp(-((x + q * T - t[k]) ** 2) / (2 * sigma**2)) for q in range(-2, 3))
        pi += alpha[k] * dens / dens.sum()
    assert abs(pi.sum() - 1) < 1e-12
    brute = np.sum(pi * np.exp(2j * np.pi * j * x / T))
    phi = oracle_mod.expected_sketch(t[None, :], alpha[None, :], sigma, T, j)[0, j - 1]
    assert abs(phi - brute) < 1e-13


def test_E3_special_cases(oracle_mod):
    """E3: sigma=0, K=1, alpha=1, t=T/4 -> Phi_1 = i; alpha=0 -> 0; |Phi| <= sum alpha; permutation
    invariance over k."""
    T = 1000
    phi = oracle_mod.expected_sketch(np.array([[T / 4]]), np.array([[1.0]]), 0.0, T, 1)[0, 0]
    assert abs(phi - 1j) < 1e-15
    assert np.all(oracle_mod.expected_sketch(np.array([[10.0, 20.0]]), np.zeros((1, 2)), 3.0, T, 5) == 0)
    rng = np.random.default_rng(5)
    t = rng.uniform(0, T, (50, 3))
    a = rng.uniform(0, 0.3, (50, 3))
    p1 = oracle_mod.expected_sketch(t, a, 2.0, T, 16)
    assert np.all(np.abs(p1) <= a.sum(1)[:, None] + 1e-15)
    perm = [2, 0, 1]
    np.testing.assert_allclose(oracle_mod.expected_sketch(t[:, perm], a[:, perm], 2.0, T, 16), p1, atol=1e-15)
    # periodic in t (reading A16)
    np.testing.assert_allclose(oracle_mod.expected_sketch(t + T, a, 2.0, T, 16), p1, atol=1e-12)


# ------------------------------------------------------ loss + gradient, Eq. (6)/(8)
def _loss_only(oracle_mod, z, t, a, sigma, T, m):
    return oracle_mod.sketch_grad(z, t, a, sigma, T, m)[2]


def test_G1_zero_gradient_at_truth(oracle_mod):
    """G1: the gradient vanishes at the true parameters of a noiseless sketch (Eq. 6 minimum)."""
    rng = np.random.default_rng(6)
    T, sigma, m, K = 8192, 6.0, 32, 3
    t = rng.uniform(0, T, (20, K))
    a = rng.uniform(0.05, 0.3, (20, K))
    z = oracle_mod.expected_sketch(t, a, sigma, T, m)
    gt, ga, L = oracle_mod.sketch_grad(z, t, a, sigma, T, m)
    assert np.abs(gt).max() < 1e-13 and np.abs(ga).max() < 1e-13 and np.abs(L).max() < 1e-28


def test_G2_finite_differences(oracle_mod):
    """G2: analytic gradient matches central finite differences of the loss,
    including SURVEY §8(c)'s instance (dL/dt_1 = 3.7107665e-4)."""
    T, sigma, m = 2500, 3.0, 5
    t = np.array([[300.25, 410.5]])
    a = np.array([[0.3, 0.2]])
    j = np.arange(1, m + 1)
    z = (0.1 * j - 0.05j * j)[None, :]
    gt, ga, L = oracle_mod.sketch_grad(z, t, a, sigma, T, m)
    assert abs(gt[0, 0] - 3.7107665e-4) < 1e-10
    rng = np.random.default_rng(8)
    cases = [(z, t, a, T, sigma, m)]
    for _ in range(6):
        K = rng.integers(1, 4)
        TT = int(rng.choice([1024, 4613, 8192]))
        mm = int(rng.integers(1, 12))
        tt = rng.uniform(0, TT, (1, K))
        aa = rng.uniform(0.05, 1, (1, K))
        zz = (rng.normal(size=(1, mm)) + 1j * rng.normal(size=(1, mm))) * 0.3
        cases.append((zz, tt, aa, TT, float(rng.uniform(0, 6)), mm))
    h = 1e-6
    for zz, tt, aa, TT, sg, mm in cases:
        gt, ga, _ = oracle_mod.sketch_grad(zz, tt, aa, sg, TT, mm)
        for k in range(tt.shape[1]):
            e = np.zeros_like(tt)
            e[0, k] = h
            fd_t = (_loss_only(oracle_mod, zz, tt + e, aa, sg, TT, mm) - _loss_only(oracle_mod, zz, tt - e, aa, sg, TT, mm))[0] / (2 * h)
            fd_a = (_loss_only(oracle_mod, zz, tt, aa + e, sg, TT, mm) - _loss_only(oracle_mod, zz, tt, aa - e, sg, TT, mm))[0] / (2 * h)
            assert abs(fd_t - gt[0, k]) <= 1e-6 * abs(gt[0, k]) + 1e-9
            assert abs(fd_a - ga[0, k]) <= 1e-6 * abs(ga[0, k]) + 1e-9


def test_G3_k1_closed_form(oracle_mod):
    """G3: K=1 with z = Phi(t*, alpha*), Delta = t - t*:
    L = sum_j h_j^2 (a*^2 + a^2 - 2 a a* cos w_j Delta); g_t = 2 a a* sum w_j h_j^2 sin w_j Delta;
    g_a = 2 sum h_j^2 (a - a* cos w_j Delta).  Worked values: SURVEY §8(c) G3 (C1-like)."""
    with open(os.path.join(GOLDEN, "g3_k1_closed_form.json")) as f:
        g = json.load(f)
    T, sigma, m = g["T"], g["sigma"], g["m"]
    for (ts, as_, t, a) in [(g["t_star"], g["alpha_star"], g["t"], g["alpha"]), (4000.0, 0.7, 3990.5, 0.2)]:
        z = oracle_mod.expected_sketch(np.array([[ts]]), np.array([[as_]]), sigma, T, m)
        gt, ga, L = oracle_mod.sketch_grad(z, np.array([[t]]), np.array([[a]]), sigma, T, m)
        w, h = _hhat(sigma, T, m)
        d = t - ts
        Lc = np.sum(h**2 * (as_**2 + a**2 - 2 * a * as_ * np.cos(w * d)))
        gtc = 2 * a * as_ * np.sum(w * h**2 * np.sin(w * d))
        gac = 2 * np.sum(h**2 * (a - as_ * np.cos(w * d)))
        assert abs(L[0] - Lc) <= 1e-13 * abs(Lc) + 1e-16
        assert abs(gt[0, 0] - gtc) <= 1e-13 * abs(gtc) + 1e-16
        assert abs(ga[0, 0] - gac) <= 1e-13 * abs(gac) + 1e-16
    z = oracle_mod.expected_sketch(np.array([[g["t_star"]]]), np.array([[g["alpha_star"]]]), sigma, T, m)
    gt, ga, L = oracle_mod.sketch_grad(z, np.array([[g["t"]]]), np.array([[g["alpha"]]]), sigma, T, m)
    assert abs(L[0] - g["loss"]) < 1e-14
    assert abs(gt[0, 0] - g["grad_t"]) < 1e-14
    assert abs(ga[0, 0] - g["grad_alpha"]) < 1e-14


def test_G4_zero_sketch(oracle_mod):
    """G4: z = 0, K=1, alpha=1, sigma=0 -> L = m, g_alpha = 2m, g_t = 0 (S:97 without the n weight)."""
    for m in (1, 4, 10, 64):
        gt, ga, L = oracle_mod.sketch_grad(np.zeros((1, m)), np.array([[123.4]]), np.array([[1.0]]), 0.0, 8192, m)
        assert abs(L[0] - m) < 1e-12 and abs(ga[0, 0] - 2 * m) < 1e-12 and abs(gt[0, 0]) < 1e-12


def test_G5_alpha_gradient_is_linear_least_squares(oracle_mod):
    """G5: g_alpha is affine in alpha and vanishes at alpha_LS = sum h Re(conj(p) z) / sum h^2 (K=1)."""
    rng = np.random.default_rng(9)
    T, sigma, m = 4613, 5.0, 10
    z = (rng.normal(size=(1, m)) + 1j * rng.normal(size=(1, m))) * 0.2
    t = np.array([[1234.56]])
    w, h = _hhat(sigma, T, m)
    p = np.exp(1j * w * t[0, 0])
    a_ls = np.sum(h * np.real(np.conj(p) * z[0])) / np.sum(h**2)
    g = [oracle_mod.sketch_grad(z, t, np.array([[a]]), sigma, T, m)[1][0, 0] for a in (a_ls, 0.0, 1.0)]
    assert abs(g[0]) < 1e-14
    assert abs((g[2] - g[1]) - 2 * np.sum(h**2)) < 1e-13  # slope 2 sum h^2


def test_G6_invariances(oracle_mod):
    """G6: alpha_k = 0 -> g_t,k = 0 exactly; t -> t+T changes nothing; (t+s, z_j e^{i w_j s})
    leaves L and g unchanged."""
    rng = np.random.default_rng(10)
    T, sigma, m, K = 2500, 3.0, 20, 2
    t = rng.uniform(0, T, (10, K))
    a = rng.uniform(0.1, 1, (10, K))
    a[:, 1] = 0.0
    z = (rng.normal(size=(10, m)) + 1j * rng.normal(size=(10, m))) * 0.2
    gt, ga, L = oracle_mod.sketch_grad(z, t, a, sigma, T, m)
    assert np.all(gt[:, 1] == 0.0)
    gt2, ga2, L2 = oracle_mod.sketch_grad(z, t + T, a, sigma, T, m)
    np.testing.assert_allclose(gt2, gt, atol=1e-12)
    np.testing.assert_allclose(L2, L, atol=1e-13)
    s = 37.3
    w, _ = _hhat(sigma, T, m)
    gt3, ga3, L3 = oracle_mod.sketch_grad(z * np.exp(1j * w * s)[None, :], t + s, a, sigma, T, m)
    np.testing.assert_allclose(gt3, gt, atol=1e-12)
    np.testing.assert_allclose(ga3, ga, atol=1e-12)
    np.testing.assert_allclose(L3, L, atol=1e-13)


# --------------------------------------------------------------- phase index (B1)
def test_B1_phase_index_edges(oracle_mod):
    """B1: r = (j x) mod T at the edge values of SURVEY §8(c)."""
    for T, x, j, r in [(4613, 4612, 10, 4603), (8192, 8191, 32, 8160), (65536, 65535, 64, 65472),
                       (65535, 65534, 64, 65471), (1024, 1023, 4, 1020), (2500, 1250, 20, 0)]:
        assert oracle_mod.phase_index(np.array([x]), T, j)[0, j - 1] == r


# -------------------------------------------------------- update rule (reading A13)
def test_update_is_diagonal_gauss_newton(oracle_mod):
    """A13 update: with eta = 1 the alpha step lands exactly on the K=1 linear least-squares
    solution, and the t step is the Gauss-Newton step (t* recovered to O(Delta^3))."""
    T, sigma, m = 4613, 5.0, 10
    ts, as_ = 2000.0, 0.6
    z = oracle_mod.expected_sketch(np.array([[ts]]), np.array([[as_]]), sigma, T, m)
    t = np.array([[ts + 0.05]])
    a = np.array([[as_]])
    gt, ga, _ = oracle_mod.sketch_grad(z, t, a, sigma, T, m)
    tn, an = oracle_mod.descent_update(t, a, gt, ga, sigma, T, m, eta=1.0)
    assert abs(tn[0, 0] - ts) < 1e-5
    w, h = _hhat(sigma, T, m)
    p = np.exp(1j * w * t[0, 0])
    a_ls = np.sum(h * np.real(np.conj(p) * z[0])) / np.sum(h**2)
    assert abs(an[0, 0] - a_ls) < 1e-14
    # clamps and wrap: a huge gradient moves t by exactly T/(4m) and wraps into [0, T)
    tn, an = oracle_mod.descent_update(np.array([[1.0]]), np.array([[0.5]]), np.array([[1e9]]), np.array([[1e9]]),
                                       sigma, T, m, eta=0.5)
    assert abs(tn[0, 0] - (1.0 - T / (4 * m) + T)) < 1e-9 and an[0, 0] == 0.0


# ------------------------------------------- NEXT-3 initialisation (A18-A20)
def _dirichlet(phi, m):
    """sum_{l=1..m} cos(l phi) in closed form (phi = 0 -> m)."""
    phi = np.asarray(phi, dtype=np.float64)
    out = np.full(phi.shape, float(m))
    nz = np.abs(np.sin(phi / 2)) > 1e-12
    out[nz] = np.sin(m * phi[nz] / 2) * np.cos((m + 1) * phi[nz] / 2) / np.sin(phi[nz] / 2)
    return out


@pytest.mark.parametrize("T,m,N", [(1024, 4, 1024), (4613, 10, 4613), (8192, 32, 256), (100, 7, 25)])
def test_BP1_single_photon_dirichlet(oracle_mod, T, m, N):
    """BP1: one photon at x, delta IRF -> g(t) is the Dirichlet kernel
    sum_l cos(omega_l (x - t)) in closed form; its maximum m sits at t = x."""
    x = (37 * T) // 100
    z = oracle_mod.sketch(np.array([x], np.uint16), np.array([0, 1], np.uint32), T, m)
    g = oracle_mod.backproject(z, 0.0, T, N)[0]
    tn = np.arange(N) * T / N
    np.testing.assert_allclose(g, _dirichlet(2 * np.pi * (x - tn) / T, m), atol=1e-11)
    if (x * N) % T == 0:
        assert np.argmax(g) == x * N // T and abs(g.max() - m) < 1e-12


def test_BP2_coefficients_recovered_by_grid_dft(oracle_mod):
    """BP2: for N > 2m the grid values determine the coefficients: (2/N) sum_n g_n e^{+i omega_l t_n}
    = hhat_l z_l (discrete orthogonality) — fixes the sign of the exponent and the hhat weight."""
    rng = np.random.default_rng(3)
    T, m, N, sigma = 2500, 20, 64, 3.0
    z = (rng.normal(size=m) + 1j * rng.normal(size=m))[None, :]
    g = oracle_mod.backproject(z, sigma, T, N)[0]
    w, h = _hhat(sigma, T, m)
    tn = np.arange(N) * T / N
    rec = np.array([(2.0 / N) * np.sum(g * np.exp(1j * wl * tn)) for wl in w])
    np.testing.assert_allclose(rec, h * z[0], atol=1e-12)


def test_BP3_bound_and_shift(oracle_mod, inputs_mod):
    """BP3: |g| <= sum_l hhat_l |z_l| (triangle inequality); shifting every photon by
    s = k T/N bins shifts g by k grid points."""
    T, m, N, sigma = 4096, 10, 512, 4.0
    bins, offs = inputs_mod.random_csr(npix=20, T=T, max_n=400, seed=5)
    z = oracle_mod.sketch(bins, offs, T, m)
    g = oracle_mod.backproject(z, sigma, T, N)
    _, h = _hhat(sigma, T, m)
    assert np.all(np.abs(g) <= np.sum(h * np.abs(z), axis=1)[:, None] + 1e-12)
    k = 13
    zs = oracle_mod.sketch(((bins.astype(np.int64) + k * T // N) % T).astype(np.uint16), offs, T, m)
    np.testing.assert_allclose(oracle_mod.backproject(zs, sigma, T, N), np.roll(g, k, axis=1), atol=1e-9)


def test_ID_greedy_picks(oracle_mod):
    """ID: single photon -> its bin; two photons farther apart than min_sep -> both,
    sorted; closer than min_sep -> one peak (a further pick is a weak side lobe); flat zero
    sketch -> none, unfilled slots per A14."""
    T, m, N = 1024, 16, 1024
    def picks(xs, K, min_sep, weights=None):
        lists = np.array(xs, np.uint16)
        z = oracle_mod.sketch(lists, np.array([0, len(xs)], np.uint32), T, m)
        g = oracle_mod.backproject(z, 0.0, T, N)
        return oracle_mod.init_depths(g, 0.0, T, m, K, min_sep)
    t, gv, a, c = picks([300], 1, 10)
    assert c[0] == 1 and t[0, 0] == 300.0 and abs(gv[0, 0] - m) < 1e-12 and a[0, 0] == 1.0
    t, gv, a, c = picks([700, 200], 2, 50)
    assert c[0] == 2 and abs(t[0, 0] - 200) <= 1 and abs(t[0, 1] - 700) <= 1  # within one grid step
    t, gv, a, c = picks([500, 520], 2, 50)  # one merged peak; the second pick is a side lobe
    main = int(np.argmax(gv[0]))
    assert 490 <= t[0, main] <= 530 and c[0] == 2
    assert gv[0, 1 - main] < 0.3 * gv[0, main] and abs(t[0, 1] - t[0, 0]) >= 50
    t, gv, a, c = picks([500, 520], 1, 50)
    assert c[0] == 1 and 490 <= t[0, 0] <= 530
    g0 = np.zeros((1, N))
    t, gv, a, c = oracle_mod.init_depths(g0, 0.0, T, m, 3, 10)
    assert c[0] == 0 and np.all(a == 0) and np.all(t == T / 2)


def test_IK_closed_form_k1(oracle_mod):
    """IK: single photon at v -> v; noiseless K=1 sketch at t = 1000, T = 4613,
    sigma = 10 -> 1000 within 1e-9 and alpha recovered (S:108 least squares); z = 0 -> 0."""
    T = 4613
    z = oracle_mod.sketch(np.array([1234], np.uint16), np.array([0, 1], np.uint32), T, 5)
    t, a = oracle_mod.init_k1(z, 0.0, T)
    assert abs(t[0] - 1234) < 1e-9 and abs(a[0] - 1) < 1e-12
    z = oracle_mod.expected_sketch(np.array([[1000.0]]), np.array([[0.37]]), 10.0, T, 10)
    t, a = oracle_mod.init_k1(z, 10.0, T)
    assert abs(t[0] - 1000.0) < 1e-9 and abs(a[0] - 0.37) < 1e-12
    z = oracle_mod.expected_sketch(np.array([[4612.75]]), np.array([[0.5]]), 3.0, T, 4)
    t, a = oracle_mod.init_k1(z, 3.0, T)
    assert abs(t[0] - 4612.75) < 1e-9 and 0 <= t[0] < T
    t, a = oracle_mod.init_k1(np.zeros((2, 4), complex), 1.0, T)
    assert np.all(t == 0) and np.all(a == 0)


# ------------------------------------------------- NEXT-4 streaming acquisition
def test_M1_merge_equals_sketch_of_concatenation(oracle_mod):
    """M1: merge of the sketches of two disjoint lists = sketch of the concatenation
    (the mean property of Eq. (3)); merge with an empty sketch is the identity; commutative;
    the online update of P:65 is the n_b = 1 case (photon at 0 then T/2 -> z_1 = 0)."""
    rng = np.random.default_rng(11)
    T, m = 4613, 10
    la = [rng.integers(0, T, rng.integers(0, 50)) for _ in range(40)]
    lb = [rng.integers(0, T, rng.integers(0, 50)) for _ in range(40)]
    def csr(lists):
        offs = np.zeros(len(lists) + 1, np.uint32)
        offs[1:] = np.cumsum([len(l) for l in lists])
        return np.concatenate(lists).astype(np.uint16), offs
    za = oracle_mod.sketch(*csr(la), T, m)
    zb = oracle_mod.sketch(*csr(lb), T, m)
    na = np.array([len(l) for l in la], np.uint32)
    nb = np.array([len(l) for l in lb], np.uint32)
    z, n = oracle_mod.sketch_merge(za, na, zb, nb)
    zc = oracle_mod.sketch(*csr([np.concatenate([a, b]) for a, b in zip(la, lb)]), T, m)
    np.testing.assert_allclose(z, zc, atol=1e-12)
    assert np.array_equal(n, na.astype(np.uint64) + nb)
    z2, _ = oracle_mod.sketch_merge(zb, nb, za, na)
    np.testing.assert_allclose(z2, z, atol=1e-15)
    z3, n3 = oracle_mod.sketch_merge(za, na, np.zeros_like(za), np.zeros_like(na))
    assert np.array_equal(z3, za) and np.array_equal(n3, na)
    T2 = 100
    z0 = oracle_mod.sketch(np.array([0], np.uint16), np.array([0, 1], np.uint32), T2, 1)
    zh = oracle_mod.sketch(np.array([50], np.uint16), np.array([0, 1], np.uint32), T2, 1)
    zz, nn = oracle_mod.sketch_merge(z0, np.array([1], np.uint32), zh, np.array([1], np.uint32))
    assert abs(zz[0, 0]) < 1e-15 and nn[0] == 2


def test_BK1_bucketing_is_a_stable_sort(oracle_mod):
    """BK1 (A21): the CSR built from an unsorted event stream equals numpy's stable argsort by
    pixel (an independent library primitive); out-of-range pixels are dropped and counted."""
    rng = np.random.default_rng(4)
    npix, nev = 300, 20000
    pix = rng.integers(0, npix + 5, nev).astype(np.uint32)
    bins = rng.integers(0, 4096, nev).astype(np.uint16)
    offs, out, dropped = oracle_mod.bucket_events(pix, bins, npix)
    keep = pix < npix
    order = np.argsort(pix[keep], kind="stable")
    assert np.array_equal(out, bins[keep][order]) and dropped == int((~keep).sum())
    assert np.array_equal(offs, np.concatenate([[0], np.cumsum(np.bincount(pix[keep], minlength=npix))]))
