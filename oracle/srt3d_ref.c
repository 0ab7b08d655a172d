/*
 * ORACLE for the SRT3D hot path — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU implementation of what the CUDA
 * path computes.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * source, header, table or constant generator with the CUDA path under
 * paper_2203_00952_b200/ (and includes none of it).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n.
 * Readings of the paper (A1..A17) are listed in DESIGN.md §3.
 *
 *   srt3d_ref_sketch           Eq. (3), with the frequency scheme
 *                              omega_l = 2*pi*l/T, l = 1..m.
 *   srt3d_ref_expected_sketch  Eq. (4), with a Gaussian IRF
 *                              hhat(w) = exp(-sigma^2 w^2 / 2) (BASELINE.json
 *                              north_star) and the background term, which is
 *                              exactly 0 at omega_l (reading A4).
 *   srt3d_ref_sketch_grad      Eq. (6)/(8) data term with W = I (P:81, P:99,
 *                              P:101), unweighted by n (reading A1), and its
 *                              analytic gradient in t_k and alpha_k.
 *   srt3d_ref_phase_index      the integer phase index r = (j*x) mod T that
 *                              omega_j * x_p reduces to (P:61 + P:84).
 *   srt3d_ref_descent_update   the harness update rule (reading A13).
 *   srt3d_ref_backproject      NEXT-3 matched-filter backprojection
 *                              g(t) = Re sum_l z_l conj(hhat_l) e^{-i omega_l t}
 *                              on the grid t_i = i T / N (A18).
 *   srt3d_ref_init_depths      NEXT-3 greedy pick of up to K local maxima of
 *                              g with a minimum circular separation (
 *                              A19).
 *   srt3d_ref_init_k1          NEXT-3 K = 1 closed form: depth from the phase
 *                              of z_1, intensity by K = 1 least squares
 *                              (A20).
 *   srt3d_ref_sketch_merge     NEXT-4 count-weighted mean of two sketches
 *                              (the online update of P:65).
 *   srt3d_ref_bucket_events    NEXT-4 stable counting sort of an unsorted
 *                              (pixel, bin) event stream into the CSR frame
 *                              srt3d_ref_sketch consumes (A21).
 *
 * Everything is computed in double precision with the textbook formula, in
 * the order the definition states; OpenMP only splits independent pixels.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define REF_OK 0
#define REF_EINVAL (-1)
#define REF_ENOMEM (-2)

/* Eq. (3): z_j = (1/n) sum_p exp(i * omega_j * x_p), omega_j = 2*pi*j/T.
 * mode 0 ("exact-index"): omega_j * x_p is reduced exactly as the integer
 *   r = (j * x_p) mod T (uint64), then cos/sin(2*pi*r/T) are read from a table
 *   filled with libm cos/sin — bit-identical to calling libm per term at the
 *   reduced argument.
 * mode 1 ("literal"): cos/sin of the unreduced argument 2*pi*j*x_p/T.
 * Empty pixel (n = 0) -> z = 0 (reading A10).
 * z is [npix][m][2] (re, im), row-major.  Photons of pixel i are
 * bins[offsets[i] .. offsets[i+1]).  Returns 0 or REF_EINVAL / REF_ENOMEM. */
int srt3d_ref_sketch(const uint16_t* bins, const uint32_t* offsets, int64_t npix,
                     uint32_t T, uint32_t m, int mode, double* z) {
  if (T < 1 || m < 1 || npix < 0) return REF_EINVAL;
  double* ctab = NULL;
  double* stab = NULL;
  if (mode == 0) {
    ctab = (double*)malloc(sizeof(double) * T);
    stab = (double*)malloc(sizeof(double) * T);
    if (!ctab || !stab) { free(ctab); free(stab); return REF_ENOMEM; }
    for (uint32_t r = 0; r < T; r++) {
      double phi = 2.0 * M_PI * (double)r / (double)T;
      ctab[r] = cos(phi);
      stab[r] = sin(phi);
    }
  }
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < npix; i++) {
    uint64_t beg = offsets[i], end = offsets[i + 1];
    uint64_t n = end - beg;
    double* zi = z + (size_t)i * m * 2;
    for (uint32_t j = 1; j <= m; j++) {
      double sre = 0.0, sim = 0.0;
      for (uint64_t p = beg; p < end; p++) {
        uint64_t x = bins[p];
        if (mode == 0) {
          uint64_t r = ((uint64_t)j * x) % (uint64_t)T;
          sre += ctab[r];
          sim += stab[r];
        } else {
          double phi = 2.0 * M_PI * (double)j * (double)x / (double)T;
          sre += cos(phi);
          sim += sin(phi);
        }
      }
      if (n == 0) {
        zi[2 * (j - 1)] = 0.0;
        zi[2 * (j - 1) + 1] = 0.0;
      } else {
        zi[2 * (j - 1)] = sre / (double)n;
        zi[2 * (j - 1) + 1] = sim / (double)n;
      }
    }
  }
  free(ctab);
  free(stab);
  return REF_OK;
}

/* r[p][j-1] = (j * x_p) mod T for j = 1..m: the integer phase index of
 * omega_j * x_p = 2*pi*j*x_p/T. */
int srt3d_ref_phase_index(const uint16_t* bins, int64_t n, uint32_t T, uint32_t m, uint32_t* r) {
  if (T < 1 || m < 1 || n < 0) return REF_EINVAL;
  for (int64_t p = 0; p < n; p++)
    for (uint32_t j = 1; j <= m; j++)
      r[(size_t)p * m + (j - 1)] = (uint32_t)(((uint64_t)j * (uint64_t)bins[p]) % (uint64_t)T);
  return REF_OK;
}

/* Eq. (4) at omega_j = 2*pi*j/T with hhat(w) = exp(-sigma^2 w^2/2):
 *   Phi_j = sum_k alpha_k * hhat(omega_j) * exp(i * omega_j * t_k)
 *           + alpha_0 * CF_uniform(omega_j),   CF_uniform(omega_j) = 0.
 * t, alpha are [npix][K] double (the GPU's fp32 values widened exactly, or
 * exact doubles for the pins); z is [npix][m][2] double. */
int srt3d_ref_expected_sketch(const double* t, const double* alpha, int64_t npix, uint32_t K,
                              double sigma, uint32_t T, uint32_t m, double* z) {
  if (T < 1 || m < 1 || K < 1 || npix < 0 || !(sigma >= 0.0)) return REF_EINVAL;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < npix; i++) {
    for (uint32_t j = 1; j <= m; j++) {
      double omega = 2.0 * M_PI * (double)j / (double)T;
      double hhat = exp(-sigma * sigma * omega * omega / 2.0);
      double re = 0.0, im = 0.0;
      for (uint32_t k = 0; k < K; k++) {
        double tk = t[(size_t)i * K + k];
        double ak = alpha[(size_t)i * K + k];
        re += ak * hhat * cos(omega * tk);
        im += ak * hhat * sin(omega * tk);
      }
      z[((size_t)i * m + (j - 1)) * 2] = re;
      z[((size_t)i * m + (j - 1)) * 2 + 1] = im;
    }
  }
  return REF_OK;
}

/* Loss and gradient of the per-pixel data term with W = I,
 * unweighted by n (reading A1):
 *   r_j   = z_j - Phi_j(theta)
 *   L     = sum_j |r_j|^2
 *   dL/dalpha_k = -2 sum_j Re( conj(r_j) * dPhi_j/dalpha_k ),
 *                 dPhi_j/dalpha_k = hhat_j exp(i omega_j t_k)
 *   dL/dt_k     = -2 sum_j Re( conj(r_j) * dPhi_j/dt_k ),
 *                 dPhi_j/dt_k = i omega_j alpha_k hhat_j exp(i omega_j t_k)
 * (chain rule of |.|^2; t in bins, omega in rad/bin).  z is [npix][m][2],
 * t and alpha [npix][K], all double (for parity: the fp32 values the GPU
 * consumed, widened exactly); outputs are double.
 * loss may be NULL. */
int srt3d_ref_sketch_grad(const double* z, const double* t, const double* alpha, int64_t npix,
                          uint32_t K, double sigma, uint32_t T, uint32_t m,
                          double* grad_t, double* grad_alpha, double* loss) {
  if (T < 1 || m < 1 || K < 1 || npix < 0 || !(sigma >= 0.0)) return REF_EINVAL;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < npix; i++) {
    double L = 0.0;
    for (uint32_t k = 0; k < K; k++) {
      grad_t[(size_t)i * K + k] = 0.0;
      grad_alpha[(size_t)i * K + k] = 0.0;
    }
    for (uint32_t j = 1; j <= m; j++) {
      double omega = 2.0 * M_PI * (double)j / (double)T;
      double hhat = exp(-sigma * sigma * omega * omega / 2.0);
      /* Phi_j */
      double phre = 0.0, phim = 0.0;
      for (uint32_t k = 0; k < K; k++) {
        double tk = t[(size_t)i * K + k];
        double ak = alpha[(size_t)i * K + k];
        phre += ak * hhat * cos(omega * tk);
        phim += ak * hhat * sin(omega * tk);
      }
      double rre = z[((size_t)i * m + (j - 1)) * 2] - phre;
      double rim = z[((size_t)i * m + (j - 1)) * 2 + 1] - phim;
      L += rre * rre + rim * rim;
      for (uint32_t k = 0; k < K; k++) {
        double tk = t[(size_t)i * K + k];
        double ak = alpha[(size_t)i * K + k];
        double pre = cos(omega * tk), pim = sin(omega * tk);
        /* dPhi/dalpha_k = hhat * p ; Re(conj(r) * hhat * p) */
        double da_re = hhat * pre, da_im = hhat * pim;
        grad_alpha[(size_t)i * K + k] += -2.0 * (rre * da_re + rim * da_im);
        /* dPhi/dt_k = i * omega * ak * hhat * p = omega*ak*hhat*(-pim + i pre) */
        double dt_re = -omega * ak * hhat * pim, dt_im = omega * ak * hhat * pre;
        grad_t[(size_t)i * K + k] += -2.0 * (rre * dt_re + rim * dt_im);
      }
    }
    if (loss) loss[i] = L;
  }
  return REF_OK;
}

/* Harness descent update (reading A13; "data_step"), in fp64:
 *   t_k     -= clamp(eta * g_t,k / (2 * max(alpha_k, 0.05)^2 * sum_j omega_j^2 hhat_j^2), +-T/(4m)),
 *              then wrapped into [0, T)
 *   alpha_k  = clamp(alpha_k - eta * g_alpha,k / (2 * sum_j hhat_j^2), 0, 1)
 * t, alpha are updated in place (double). */
int srt3d_ref_descent_update(double* t, double* alpha, const double* grad_t, const double* grad_alpha,
                             int64_t npix, uint32_t K, double sigma, uint32_t T, uint32_t m, double eta) {
  if (T < 1 || m < 1 || K < 1 || npix < 0 || !(sigma >= 0.0)) return REF_EINVAL;
  double sw2h2 = 0.0, sh2 = 0.0;
  for (uint32_t j = 1; j <= m; j++) {
    double omega = 2.0 * M_PI * (double)j / (double)T;
    double hhat = exp(-sigma * sigma * omega * omega / 2.0);
    sw2h2 += omega * omega * hhat * hhat;
    sh2 += hhat * hhat;
  }
  double maxstep = (double)T / (4.0 * (double)m);
  for (int64_t q = 0; q < npix * (int64_t)K; q++) {
    double a = alpha[q];
    double am = a > 0.05 ? a : 0.05;
    double step = eta * grad_t[q] / (2.0 * am * am * sw2h2);
    if (step > maxstep) step = maxstep;
    if (step < -maxstep) step = -maxstep;
    double tn = t[q] - step;
    tn = fmod(tn, (double)T);
    if (tn < 0.0) tn += (double)T;
    t[q] = tn;
    double an = a - eta * grad_alpha[q] / (2.0 * sh2);
    if (an < 0.0) an = 0.0;
    if (an > 1.0) an = 1.0;
    alpha[q] = an;
  }
  return REF_OK;
}

/* ---- NEXT-3: pixelwise initialisation (A18-A20) ---- */

/* g[i][n] = Re sum_{l=1..m} z_l * hhat_l * exp(-i * omega_l * t_n), t_n = n*T/N,
 * omega_l = 2*pi*l/T, hhat real (Gaussian, reading A5) so conj(hhat) = hhat.
 * The phase omega_l * t_n = 2*pi*l*n/N is reduced exactly as (l*n) mod N. */
int srt3d_ref_backproject(const double* z, int64_t npix, double sigma, uint32_t T, uint32_t m,
                          uint32_t N, double* g) {
  if (T < 1 || m < 1 || N < 1 || npix < 0 || !(sigma >= 0.0)) return REF_EINVAL;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < npix; i++) {
    for (uint32_t n = 0; n < N; n++) {
      double acc = 0.0;
      for (uint32_t l = 1; l <= m; l++) {
        double omega = 2.0 * M_PI * (double)l / (double)T;
        double hhat = exp(-sigma * sigma * omega * omega / 2.0);
        uint64_t r = ((uint64_t)l * (uint64_t)n) % (uint64_t)N;
        double ph = -2.0 * M_PI * (double)r / (double)N;
        double zre = z[((size_t)i * m + (l - 1)) * 2], zim = z[((size_t)i * m + (l - 1)) * 2 + 1];
        /* Re((zre + i zim) * hhat * (cos ph + i sin ph)) */
        acc += hhat * (zre * cos(ph) - zim * sin(ph));
      }
      g[(size_t)i * N + n] = acc;
    }
  }
  return REF_OK;
}

/* Greedy initial depths from g (one pixel row of N values, grid t_n = n*T/N):
 *   candidates: n with g_n > 0, g_n > g_{n-1} and g_n >= g_{n+1} (circular, N >= 3);
 *   K times: the candidate with the largest g (ties: smallest n) whose circular
 *   grid distance d to every earlier pick satisfies d*T >= min_sep*N.
 * Outputs, sorted by depth: t_out[k] = n_k*T/N, g_out[k] = g_{n_k}, and
 * alpha_out[k] = clamp(g_{n_k} / sum_l hhat_l^2, 0, 1); count[i] = picks.
 * Unfilled slots (reading A14): t = (t_first + T/2) mod T (T/2 if none),
 * g = alpha = 0.  Input g is the fp64 backprojection above. */
int srt3d_ref_init_depths(const double* g, int64_t npix, double sigma, uint32_t T, uint32_t m, uint32_t N,
                          uint32_t K, uint32_t min_sep, double* t_out, double* g_out, double* alpha_out,
                          int32_t* count) {
  if (T < 1 || m < 1 || N < 3 || K < 1 || npix < 0 || !(sigma >= 0.0)) return REF_EINVAL;
  double sh2 = 0.0;
  for (uint32_t l = 1; l <= m; l++) {
    double omega = 2.0 * M_PI * (double)l / (double)T;
    double hhat = exp(-sigma * sigma * omega * omega / 2.0);
    sh2 += hhat * hhat;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < npix; i++) {
    const double* gi = g + (size_t)i * N;
    uint32_t pick[64];
    uint32_t c = 0;
    for (uint32_t k = 0; k < K && k < 64; k++) {
      int64_t best = -1;
      for (uint32_t n = 0; n < N; n++) {
        double gp = gi[(n + N - 1) % N], gn = gi[(n + 1) % N];
        if (!(gi[n] > 0.0 && gi[n] > gp && gi[n] >= gn)) continue;
        int ok = 1;
        for (uint32_t q = 0; q < c; q++) {
          uint32_t d = n > pick[q] ? n - pick[q] : pick[q] - n;
          if (N - d < d) d = N - d;
          if ((uint64_t)d * T < (uint64_t)min_sep * N) ok = 0;
        }
        if (ok && (best < 0 || gi[n] > gi[best])) best = n;
      }
      if (best < 0) break;
      pick[c++] = (uint32_t)best;
    }
    /* sort picks by grid index (= depth) */
    for (uint32_t a = 1; a < c; a++)
      for (uint32_t b = a; b > 0 && pick[b - 1] > pick[b]; b--) {
        uint32_t tmp = pick[b];
        pick[b] = pick[b - 1];
        pick[b - 1] = tmp;
      }
    double tfirst = c ? (double)pick[0] * (double)T / (double)N : 0.0;
    for (uint32_t k = 0; k < K; k++) {
      size_t o = (size_t)i * K + k;
      if (k < c) {
        double gv = gi[pick[k]];
        double a = gv / sh2;
        t_out[o] = (double)pick[k] * (double)T / (double)N;
        g_out[o] = gv;
        alpha_out[o] = a < 0.0 ? 0.0 : (a > 1.0 ? 1.0 : a);
      } else {
        t_out[o] = fmod(tfirst + 0.5 * (double)T, (double)T);
        g_out[o] = 0.0;
        alpha_out[o] = 0.0;
      }
    }
    count[i] = (int32_t)c;
  }
  return REF_OK;
}

/* K = 1 closed form: t = (T / 2 pi) * arg(z_1 * conj(hhat_1)) mapped into
 * [0, T) (hhat_1 > 0, so arg(z_1)); alpha = clamp(sum_l hhat_l Re(conj(e^{i omega_l t}) z_l)
 * / sum_l hhat_l^2, 0, 1), the least-squares alpha at t.  |z_1| <= 1e-12:
 * t = alpha = 0. */
int srt3d_ref_init_k1(const double* z, int64_t npix, double sigma, uint32_t T, uint32_t m, double* t_out,
                      double* alpha_out) {
  if (T < 1 || m < 1 || npix < 0 || !(sigma >= 0.0)) return REF_EINVAL;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < npix; i++) {
    double z1re = z[(size_t)i * m * 2], z1im = z[(size_t)i * m * 2 + 1];
    if (hypot(z1re, z1im) <= 1e-12) {
      t_out[i] = 0.0;
      alpha_out[i] = 0.0;
      continue;
    }
    double t = (double)T * atan2(z1im, z1re) / (2.0 * M_PI);
    if (t < 0.0) t += (double)T;
    if (t >= (double)T) t -= (double)T;
    double num = 0.0, den = 0.0;
    for (uint32_t l = 1; l <= m; l++) {
      double omega = 2.0 * M_PI * (double)l / (double)T;
      double hhat = exp(-sigma * sigma * omega * omega / 2.0);
      double zre = z[((size_t)i * m + (l - 1)) * 2], zim = z[((size_t)i * m + (l - 1)) * 2 + 1];
      /* Re(conj(cos + i sin) * z) = cos * zre + sin * zim */
      num += hhat * (cos(omega * t) * zre + sin(omega * t) * zim);
      den += hhat * hhat;
    }
    double a = num / den;
    t_out[i] = t;
    alpha_out[i] = a < 0.0 ? 0.0 : (a > 1.0 ? 1.0 : a);
  }
  return REF_OK;
}

/* ---- NEXT-4: streaming acquisition (A21) ---- */

/* z = (n_a z_a + n_b z_b) / (n_a + n_b), n = n_a + n_b per pixel;
 * n = 0 -> z = 0.  z_* are [npix][m][2]. */
int srt3d_ref_sketch_merge(const double* za, const uint32_t* na, const double* zb, const uint32_t* nb,
                           int64_t npix, uint32_t m, double* z, uint64_t* n) {
  if (m < 1 || npix < 0) return REF_EINVAL;
  for (int64_t i = 0; i < npix; i++) {
    uint64_t nn = (uint64_t)na[i] + (uint64_t)nb[i];
    n[i] = nn;
    for (uint32_t j = 0; j < 2 * m; j++) {
      size_t o = (size_t)i * 2 * m + j;
      z[o] = nn ? ((double)na[i] * za[o] + (double)nb[i] * zb[o]) / (double)nn : 0.0;
    }
  }
  return REF_OK;
}

/* Stable counting sort by pixel: offsets[i] = number of events with pixel < i
 * (offsets[npix] = kept events); bins_out lists each pixel's bins in event
 * order.  Events with pix >= npix are dropped (*dropped counts them). */
int srt3d_ref_bucket_events(const uint32_t* pix, const uint16_t* bins, uint64_t nev, int64_t npix,
                            uint32_t* offsets, uint16_t* bins_out, uint64_t* dropped) {
  if (npix < 0) return REF_EINVAL;
  uint64_t* cnt = (uint64_t*)calloc((size_t)npix + 1, sizeof(uint64_t));
  if (!cnt) return REF_ENOMEM;
  uint64_t drop = 0;
  for (uint64_t e = 0; e < nev; e++) {
    if ((int64_t)pix[e] < npix) cnt[pix[e] + 1]++;
    else drop++;
  }
  for (int64_t i = 0; i < npix; i++) cnt[i + 1] += cnt[i];
  for (int64_t i = 0; i <= npix; i++) offsets[i] = (uint32_t)cnt[i];
  for (uint64_t e = 0; e < nev; e++)
    if ((int64_t)pix[e] < npix) bins_out[cnt[pix[e]]++] = bins[e];
  *dropped = drop;
  free(cnt);
  return REF_OK;
}

/* Total photon count helper for tests (not part of the method). */
uint64_t srt3d_ref_total_photons(const uint32_t* offsets, int64_t npix) {
  return npix > 0 ? (uint64_t)offsets[npix] - (uint64_t)offsets[0] : 0;
}
