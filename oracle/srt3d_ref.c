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

/* Total photon count helper for tests (not part of the method). */
uint64_t srt3d_ref_total_photons(const uint32_t* offsets, int64_t npix) {
  return npix > 0 ? (uint64_t)offsets[npix] - (uint64_t)offsets[0] : 0;
}
