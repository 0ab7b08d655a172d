/*
 * Seeded synthetic photon-frame generator (input synthesis only; shared by the
 * oracle tests and the CUDA tests/bench).  It holds none of the method's
 * arithmetic: no sketch, no characteristic function, no loss or gradient.
 *
 * Model sampled: the mixture of Eq. (1) on the bin grid
 * {0..T-1}:
 *   - background photons uniform on {0..T-1},
 *   - signal photons of surface k from the wrapped discrete Gaussian
 *       P(x) ∝ sum_q exp(-(x + qT - t_k)^2 / (2 sigma^2)),  x in {0..T-1}
 *     (reading A8), sampled by inverse CDF over the window
 *     [floor(t)-W, ceil(t)+W], W = ceil(8 sigma)+1, then wrapped mod T;
 *     sigma = 0 puts every signal photon at round(t) mod T.
 * Photon classes are drawn categorically with weights (b, lam_1..lam_K) per
 * pixel; photon counts are Poisson(b + sum_k lam_k) (PTRS, Hörmann 1993) or a
 * fixed count.
 *
 * RNG: counter-based.  Every uniform is splitmix64-finalised from
 * (seed, stream, pixel, counter), so the frame is bit-identical for any
 * thread count ("per-pixel deterministic substream").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

typedef struct {
  uint64_t key;
  uint64_t ctr;
} rng_t;

static inline rng_t rng_make(uint64_t seed, uint64_t stream, uint64_t pixel) {
  rng_t r;
  r.key = mix64(mix64(seed ^ 0x6A09E667F3BCC908ULL) + 0x9E3779B97F4A7C15ULL * (stream + 1)) ^
          mix64(0xD1B54A32D192ED03ULL * (pixel + 1));
  r.ctr = 0;
  return r;
}
static inline uint64_t rng_u64(rng_t* r) { return mix64(r->key + 0x9E3779B97F4A7C15ULL * (++r->ctr)); }
/* uniform double in [0,1) with 53 random bits */
static inline double rng_unif(rng_t* r) { return (double)(rng_u64(r) >> 11) * (1.0 / 9007199254740992.0); }
/* uniform integer in [0, n) by 64x64->128 multiply (bias < n/2^64) */
static inline uint32_t rng_below(rng_t* r, uint32_t n) {
  return (uint32_t)(((unsigned __int128)rng_u64(r) * (unsigned __int128)n) >> 64);
}

/* Poisson(mu): inversion for mu < 10, PTRS (transformed rejection with
 * squeeze, Hörmann 1993) otherwise. */
static uint64_t poisson(rng_t* r, double mu) {
  if (mu <= 0.0) return 0;
  if (mu < 10.0) {
    double L = exp(-mu), p = 1.0;
    uint64_t k = 0;
    do {
      k++;
      p *= rng_unif(r);
    } while (p > L);
    return k - 1;
  }
  double slam = sqrt(mu), loglam = log(mu);
  double b = 0.931 + 2.53 * slam;
  double a = -0.059 + 0.02483 * b;
  double invalpha = 1.1239 + 1.1328 / (b - 3.4);
  double vr = 0.9277 - 3.6224 / (b - 2.0);
  for (;;) {
    double U = rng_unif(r) - 0.5;
    double V = rng_unif(r);
    double us = 0.5 - fabs(U);
    double kd = floor((2.0 * a / us + b) * U + mu + 0.43);
    if (kd < 0.0) continue;
    if (us >= 0.07 && V <= vr) return (uint64_t)kd;
    if (us < 0.013 && V > us) continue;
    double lhs = log(V) + log(invalpha) - log(a / (us * us) + b);
    double rhs = -mu + kd * loglam - lgamma(kd + 1.0);
    if (lhs <= rhs) return (uint64_t)kd;
  }
}

/* Pass 1: photon counts.  mean[i] = expected count of pixel i; if
 * fixed_n >= 0 every pixel gets exactly fixed_n photons. */
int srt3d_gen_counts(const double* mean, int64_t npix, int64_t fixed_n, uint64_t seed, uint64_t* counts) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < npix; i++) {
    if (fixed_n >= 0) {
      counts[i] = (uint64_t)fixed_n;
    } else {
      rng_t r = rng_make(seed, 1, (uint64_t)i);
      counts[i] = poisson(&r, mean[i]);
    }
  }
  return 0;
}

/* Pass 2: photon time stamps for every pixel, written at bins[offsets[i]..].
 * weights[i][0] = background weight b_i, weights[i][1+k] = lam_ik (any
 * non-negative scale; only ratios matter); t[i][k] = surface depth (bins).
 * Writes uint16 bins; T <= 65536. */
int srt3d_gen_photons(const uint32_t* offsets, int64_t npix, uint32_t K, const double* weights,
                      const float* t, double sigma, uint32_t T, uint64_t seed, uint16_t* bins) {
  if (T < 1 || T > 65536 || K < 1 || K > 16) return -1;
  const int W = (int)ceil(8.0 * sigma) + 1;
  const int L = 2 * W + 2; /* window length */
  int fail = 0;
#pragma omp parallel
  {
    double* cdf = (double*)malloc(sizeof(double) * (size_t)L * K);
    int64_t* lo = (int64_t*)malloc(sizeof(int64_t) * K);
    if (!cdf || !lo) {
#pragma omp atomic write
      fail = 1;
    }
#pragma omp for schedule(dynamic, 4)
    for (int64_t i = 0; i < npix; i++) {
      if (!cdf || !lo) continue;
      const double* wi = weights + (size_t)i * (K + 1);
      double tot = 0.0, cum[17];
      for (uint32_t c = 0; c <= K; c++) {
        tot += wi[c];
        cum[c] = tot;
      }
      /* per-surface inverse-CDF tables of the wrapped discrete Gaussian */
      for (uint32_t k = 0; k < K; k++) {
        double tk = (double)t[(size_t)i * K + k];
        double* ck = cdf + (size_t)k * L;
        lo[k] = (int64_t)floor(tk) - W;
        if (sigma > 0.0) {
          double s = 0.0;
          for (int u = 0; u < L; u++) {
            double d = (double)(lo[k] + u) - tk;
            s += exp(-d * d / (2.0 * sigma * sigma));
            ck[u] = s;
          }
          for (int u = 0; u < L; u++) ck[u] /= s;
        }
      }
      rng_t r = rng_make(seed, 2, (uint64_t)i);
      uint64_t beg = offsets[i], end = offsets[i + 1];
      for (uint64_t p = beg; p < end; p++) {
        double uc = rng_unif(&r) * tot;
        uint32_t c = 0;
        while (c < K && uc >= cum[c]) c++;
        uint32_t x;
        if (c == 0 || tot <= 0.0) {
          x = rng_below(&r, T);
        } else {
          uint32_t k = c - 1;
          int64_t u;
          if (sigma > 0.0) {
            double v = rng_unif(&r);
            const double* ck = cdf + (size_t)k * L;
            int a = 0, b = L - 1; /* first index with ck[idx] > v */
            while (a < b) {
              int mid = (a + b) >> 1;
              if (ck[mid] > v) b = mid; else a = mid + 1;
            }
            u = lo[k] + a;
          } else {
            u = (int64_t)llrint((double)t[(size_t)i * K + k]);
          }
          int64_t xm = u % (int64_t)T;
          if (xm < 0) xm += T;
          x = (uint32_t)xm;
        }
        bins[p] = (uint16_t)x;
      }
    }
    free(cdf);
    free(lo);
  }
  return fail ? -2 : 0;
}
