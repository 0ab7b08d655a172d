// C ABI of libsrt3d.so (declared in include/srt3d.h): host-side validation,
// per-call constants (fp64 on the host), launch-regime choice and error
// reporting.  Validation precedes every launch, so a failing call writes
// nothing.
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/srt3d.h"
#include "kernels.h"

namespace {

thread_local char g_err[512] = "no error";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SRT3D_ECUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

int num_sms_current() { return srt3d::num_sms_device(); }

bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

int check_tm(uint32_t T, uint32_t m) {
  if (T < 2 || T > SRT3D_MAX_T) return fail(SRT3D_EINVAL, "T=%u out of range [2, %u]", T, SRT3D_MAX_T);
  if (m < 1 || m >= T) return fail(SRT3D_EINVAL, "m=%u must satisfy 1 <= m <= T-1 (T=%u)", m, T);
  if (m > SRT3D_MAX_M) return fail(SRT3D_EUNSUPPORTED, "m=%u exceeds SRT3D_MAX_M=%u", m, SRT3D_MAX_M);
  return SRT3D_OK;
}

int check_kparams(int64_t npix, uint32_t K, float sigma, uint32_t T, uint32_t m) {
  if (npix < 0) return fail(SRT3D_EINVAL, "npix=%lld < 0", (long long)npix);
  int rc = check_tm(T, m);
  if (rc) return rc;
  if (K < 1) return fail(SRT3D_EINVAL, "K=%u < 1", K);
  if (K > SRT3D_MAX_K) return fail(SRT3D_EUNSUPPORTED, "K=%u exceeds SRT3D_MAX_K=%u", K, SRT3D_MAX_K);
  if (!std::isfinite(sigma) || sigma < 0.f) return fail(SRT3D_EINVAL, "sigma=%g must be finite and >= 0", (double)sigma);
  return SRT3D_OK;
}

// fp64 constants, rounded once
void fill_consts(srt3d::PixArgs& a, float sigma, uint32_t T, uint32_t m, float eta) {
  const double pi = 3.14159265358979323846;
  double sw2h2 = 0.0, sh2 = 0.0;
  for (int j = 0; j < srt3d::MAX_M; j++) {
    a.c.hh[j] = 0.f;
    a.c.wh[j] = 0.f;
  }
  for (uint32_t j = 1; j <= m; j++) {
    const double w = 2.0 * pi * (double)j / (double)T;
    const double h = std::exp(-(double)sigma * (double)sigma * w * w / 2.0);
    a.c.hh[j - 1] = (float)h;
    a.c.wh[j - 1] = (float)(w * h);
    sw2h2 += w * w * h * h;
    sh2 += h * h;
  }
  a.T = T;
  a.m = m;
  a.invT = 1.0 / (double)T;
  a.Tf = (float)T;
  a.invTf = (float)(1.0 / (double)T);
  a.eta = eta;
  a.upd_t_scale = (float)(1.0 / (2.0 * sw2h2));
  a.upd_a_scale = (float)(1.0 / (2.0 * sh2));
  a.max_step = (float)((double)T / (4.0 * (double)m));
}

bool pair_fits(uint32_t T) { return T <= srt3d::SO_MAX_T; }

bool hist_fits(uint32_t T, int M) { return srt3d::sketch_hist_smem(T, M) <= 227u * 1024u; }

// Lanes per pixel of a regime (0: bin-count, one CTA per pixel).
int regime_lanes(uint32_t rg) {
  switch (rg) {
    case srt3d::RG_G4:
    case srt3d::RG_G4C:
      return 4;
    case srt3d::RG_RT:
      return 2;
    case srt3d::RG_G8:
      return 8;
    case srt3d::RG_G16:
      return 16;
    case srt3d::RG_G32:
      return 32;
    default:
      return 0;
  }
}

cudaError_t launch_regime(uint32_t rg, int M, const srt3d::SketchArgs& a, cudaStream_t s, int nsm) {
  switch (rg) {
    case srt3d::RG_G4C:
      return srt3d::launch_sketch_pass(M, srt3d::SK_G4_CHEB, a, s, nsm);
    case srt3d::RG_RT:
      return srt3d::launch_sketch_routed(M, a, s, nsm);
    case srt3d::RG_TC:
      return srt3d::launch_sketch_tc(M, a, s, nsm);
    case srt3d::RG_H128:
      return srt3d::launch_sketch_hist(M, a, 128, s, nsm);
    case srt3d::RG_H256:
      return srt3d::launch_sketch_hist(M, a, 256, s, nsm);
    case srt3d::RG_H512:
      return srt3d::launch_sketch_hist(M, a, 512, s, nsm);
    default:
      return srt3d::launch_sketch_pass(M, regime_lanes(rg), a, s, nsm);
  }
}

// Regimes sketch_regime() can return for (npix, T, M, mode) at any photon
// count: it is piecewise constant in the mean photons per pixel with
// breakpoints at these means, so evaluating it there finds every candidate.
int regime_candidates(int64_t npix, uint32_t T, int M, uint32_t mode, uint32_t j0, uint32_t* out) {
  const unsigned long long np = (unsigned long long)npix;
  const unsigned long long means[] = {0, 256, 2048, 4096, T, srt3d::TC_MAX_MEAN_PER_T * T, 30000, 80000};
  int n = 0;
  for (unsigned long long mu : means) {
    const unsigned long long tot = mu * np;
    if (tot >= (1ull << 32)) continue;  // total photons < 2^32 (precondition)
    const uint32_t rg = srt3d::sketch_regime(tot, npix, T, M, mode, j0);
    bool seen = false;
    for (int i = 0; i < n; i++) seen = seen || out[i] == rg;
    if (!seen) out[n++] = rg;
  }
  return n;
}

// The sketch entry points.  have_hint: total_photons = offsets[npix] -
// offsets[0] is known on the host, so the regime is chosen here; otherwise
// every candidate regime of the pass is launched with rg_want set and each
// kernel picks itself (or exits) from the two offsets it reads on the device:
// no host read, no synchronisation, graph-capturable.  A wrong hint changes
// only the launch shape, never the result (every regime computes Eq. (3)).
int sketch_entry(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, uint32_t m, float* z,
                 bool have_hint, uint64_t total, int path, int lanes_per_pixel, void* stream) {
  if (npix < 0) return fail(SRT3D_EINVAL, "npix=%lld < 0", (long long)npix);
  int rc = check_tm(T, m);
  if (rc) return rc;
  if (path < SRT3D_PATH_AUTO || path > SRT3D_PATH_TENSOR) return fail(SRT3D_EINVAL, "path=%d unknown", path);
  if (path == SRT3D_PATH_ROUTED && lanes_per_pixel != 0 && lanes_per_pixel != 2)
    return fail(SRT3D_EINVAL, "routed path: lanes_per_pixel=%d must be 0 or 2", lanes_per_pixel);
  if (path == SRT3D_PATH_TENSOR && lanes_per_pixel != 0)
    return fail(SRT3D_EINVAL, "tensor-core path: lanes_per_pixel=%d must be 0", lanes_per_pixel);
  if (path != SRT3D_PATH_ROUTED && lanes_per_pixel != 0 && lanes_per_pixel != 4 && lanes_per_pixel != 8 &&
      lanes_per_pixel != 16 && lanes_per_pixel != 32)
    return fail(SRT3D_EINVAL, "lanes_per_pixel=%d must be 0, 4, 8, 16 or 32", lanes_per_pixel);
  if (npix == 0) return SRT3D_OK;
  if (!bins || !offsets || !z) return fail(SRT3D_ENULL, "bins/offsets/z must be non-NULL");
  if (!aligned(bins, 2) || !aligned(offsets, 4) || !aligned(z, 8))
    return fail(SRT3D_EALIGN, "bins/offsets/z must be 2/4/8-byte aligned");
  const int M0 = (int)(m < 32 ? m : 32);
  if (path == SRT3D_PATH_BINCOUNT && !hist_fits(T, M0))
    return fail(SRT3D_EUNSUPPORTED, "bin-count path needs T <= ~17000 (T=%u)", T);
  if (path == SRT3D_PATH_PAIRED && !pair_fits(T))
    return fail(SRT3D_EUNSUPPORTED, "class-sorted path needs T <= %u (T=%u)", srt3d::SO_MAX_T, T);
  if (path == SRT3D_PATH_ROUTED && !srt3d::routed_fits(T, 0))
    return fail(SRT3D_EUNSUPPORTED, "routed path needs T %% 4 == 0 and T <= %u (T=%u)", srt3d::RT_MAX_T, T);
  if (path == SRT3D_PATH_TENSOR && !srt3d::tc_fits(T))
    return fail(SRT3D_EUNSUPPORTED, "tensor-core path needs T <= %u (T=%u)", srt3d::TC_MAX_T, T);
  cudaStream_t s = (cudaStream_t)stream;
  const int nsm = num_sms_current();
  srt3d::SketchArgs a = {};
  a.bins = bins;
  a.offsets = offsets;
  a.npix = npix;
  a.T = T;
  a.mstride = m;
  a.z = z;
  for (uint32_t j0 = 0; j0 < m; j0 += 32) {
    a.j0 = j0;
    a.rg_want = srt3d::RG_NONE;
    const int M = (int)((m - j0) < 32 ? (m - j0) : 32);
    cudaError_t e = cudaSuccess;
    if (path == SRT3D_PATH_PAIRED) {
      e = srt3d::launch_sketch_pair(M, a, s, nsm);
    } else if (path == SRT3D_PATH_TENSOR) {
      e = srt3d::launch_sketch_tc(M, a, s, nsm);
    } else if (path == SRT3D_PATH_ROUTED) {
      e = j0 == 0 ? srt3d::launch_sketch_routed(M, a, s, nsm)
                  : srt3d::launch_sketch_pass(M, M >= 24 ? srt3d::SK_G4_CHEB : 4, a, s, nsm);
    } else if (path == SRT3D_PATH_DIRECT && lanes_per_pixel != 0) {
      e = srt3d::launch_sketch_pass(M, lanes_per_pixel, a, s, nsm);
    } else {
      const uint32_t mode = path == SRT3D_PATH_BINCOUNT ? srt3d::RGM_HIST
                            : (path == SRT3D_PATH_AUTO && hist_fits(T, M)) ? srt3d::RGM_AUTO
                                                                            : srt3d::RGM_DIRECT;
      a.rg_mode = mode;
      if (have_hint) {
        e = launch_regime(srt3d::sketch_regime(total, npix, T, M, mode, j0), M, a, s, nsm);
      } else {
        uint32_t cand[8];
        const int nc = regime_candidates(npix, T, M, mode, j0, cand);
        for (int i = 0; i < nc && e == cudaSuccess; i++) {
          a.rg_want = nc > 1 ? cand[i] : srt3d::RG_NONE;
          e = launch_regime(cand[i], M, a, s, nsm);
        }
      }
    }
    if (e != cudaSuccess) return cuda_fail(e, "srt3d_sketch");
  }
  return SRT3D_OK;
}

}  // namespace

extern "C" {

int srt3d_version(void) { return 100; }

const char* srt3d_last_error(void) { return g_err; }

int srt3d_sketch(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, uint32_t m, float* z,
                 void* stream) {
  return sketch_entry(bins, offsets, npix, T, m, z, false, 0, SRT3D_PATH_AUTO, 0, stream);
}

int srt3d_sketch_ex(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, uint32_t m, float* z,
                    uint64_t total_photons_hint, int path, int lanes_per_pixel, void* stream) {
  return sketch_entry(bins, offsets, npix, T, m, z, total_photons_hint != SRT3D_HINT_UNKNOWN, total_photons_hint,
                      path, lanes_per_pixel, stream);
}

int srt3d_sketch_plan(int64_t npix, uint32_t T, uint32_t m, uint64_t total_photons, int* lanes_per_pixel) {
  if (npix <= 0) return fail(SRT3D_EINVAL, "npix=%lld must be > 0", (long long)npix);
  int rc = check_tm(T, m);
  if (rc) return rc;
  const int M0 = (int)(m < 32 ? m : 32);
  const uint32_t rg = srt3d::sketch_regime(total_photons, npix, T, M0,
                                           hist_fits(T, M0) ? srt3d::RGM_AUTO : srt3d::RGM_DIRECT, 0);
  if (lanes_per_pixel) *lanes_per_pixel = regime_lanes(rg);
  return rg >= srt3d::RG_H128 ? SRT3D_PATH_BINCOUNT
         : rg == srt3d::RG_RT ? SRT3D_PATH_ROUTED
         : rg == srt3d::RG_TC ? SRT3D_PATH_TENSOR
                              : SRT3D_PATH_DIRECT;
}

int srt3d_expected_sketch(const float* t, const float* alpha, int64_t npix, uint32_t K, float sigma, uint32_t T,
                          uint32_t m, float* z, void* stream) {
  int rc = check_kparams(npix, K, sigma, T, m);
  if (rc) return rc;
  if (npix == 0) return SRT3D_OK;
  if (!t || !alpha || !z) return fail(SRT3D_ENULL, "t/alpha/z must be non-NULL");
  if (!aligned(t, 4) || !aligned(alpha, 4) || !aligned(z, 8))
    return fail(SRT3D_EALIGN, "t/alpha must be 4-byte and z 8-byte aligned");
  srt3d::PixArgs a = {};
  fill_consts(a, sigma, T, m, 0.f);
  a.t_in = t;
  a.a_in = alpha;
  a.zout = z;
  a.npix = npix;
  cudaError_t e = srt3d::launch_pixel(srt3d::PX_EXPECTED, (int)K, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_expected_sketch");
  return SRT3D_OK;
}

int srt3d_sketch_grad(const float* z, const float* t, const float* alpha, int64_t npix, uint32_t K, float sigma,
                      uint32_t T, uint32_t m, float* grad_t, float* grad_alpha, float* loss, void* stream) {
  int rc = check_kparams(npix, K, sigma, T, m);
  if (rc) return rc;
  if (npix == 0) return SRT3D_OK;
  if (!z || !t || !alpha || !grad_t || !grad_alpha) return fail(SRT3D_ENULL, "z/t/alpha/grad_t/grad_alpha must be non-NULL");
  if (!aligned(z, 8) || !aligned(t, 4) || !aligned(alpha, 4) || !aligned(grad_t, 4) || !aligned(grad_alpha, 4) ||
      (loss && !aligned(loss, 4)))
    return fail(SRT3D_EALIGN, "z must be 8-byte and t/alpha/grads/loss 4-byte aligned");
  srt3d::PixArgs a = {};
  fill_consts(a, sigma, T, m, 0.f);
  a.z = z;
  a.t_in = t;
  a.a_in = alpha;
  a.grad_t = grad_t;
  a.grad_a = grad_alpha;
  a.loss = loss;
  a.npix = npix;
  cudaError_t e = srt3d::launch_pixel(srt3d::PX_GRAD, (int)K, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_sketch_grad");
  return SRT3D_OK;
}

int srt3d_descent_update(float* t, float* alpha, const float* grad_t, const float* grad_alpha, int64_t npix,
                         uint32_t K, float sigma, uint32_t T, uint32_t m, float eta, void* stream) {
  int rc = check_kparams(npix, K, sigma, T, m);
  if (rc) return rc;
  if (!std::isfinite(eta) || eta <= 0.f) return fail(SRT3D_EINVAL, "eta=%g must be finite and > 0", (double)eta);
  if (npix == 0) return SRT3D_OK;
  if (!t || !alpha || !grad_t || !grad_alpha) return fail(SRT3D_ENULL, "t/alpha/grad_t/grad_alpha must be non-NULL");
  if (!aligned(t, 4) || !aligned(alpha, 4) || !aligned(grad_t, 4) || !aligned(grad_alpha, 4))
    return fail(SRT3D_EALIGN, "t/alpha/grads must be 4-byte aligned");
  srt3d::PixArgs a = {};
  fill_consts(a, sigma, T, m, eta);
  a.t_in = t;
  a.a_in = alpha;
  a.t_out = t;
  a.a_out = alpha;
  a.grad_t = const_cast<float*>(grad_t);
  a.grad_a = const_cast<float*>(grad_alpha);
  a.npix = npix;
  cudaError_t e = srt3d::launch_pixel(srt3d::PX_UPDATE, (int)K, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_descent_update");
  return SRT3D_OK;
}

int srt3d_sketch_grad_step(const float* z, float* t, float* alpha, int64_t npix, uint32_t K, float sigma, uint32_t T,
                           uint32_t m, float eta, float* loss, void* stream) {
  int rc = check_kparams(npix, K, sigma, T, m);
  if (rc) return rc;
  if (!std::isfinite(eta) || eta <= 0.f) return fail(SRT3D_EINVAL, "eta=%g must be finite and > 0", (double)eta);
  if (npix == 0) return SRT3D_OK;
  if (!z || !t || !alpha) return fail(SRT3D_ENULL, "z/t/alpha must be non-NULL");
  if (!aligned(z, 8) || !aligned(t, 4) || !aligned(alpha, 4) || (loss && !aligned(loss, 4)))
    return fail(SRT3D_EALIGN, "z must be 8-byte and t/alpha/loss 4-byte aligned");
  srt3d::PixArgs a = {};
  fill_consts(a, sigma, T, m, eta);
  a.z = z;
  a.t_in = t;
  a.a_in = alpha;
  a.t_out = t;
  a.a_out = alpha;
  a.loss = loss;
  a.npix = npix;
  cudaError_t e = srt3d::launch_pixel(srt3d::PX_GRAD_STEP, (int)K, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_sketch_grad_step");
  return SRT3D_OK;
}

int srt3d_fit_pixelwise(const float* z, float* t, float* alpha, int64_t npix, uint32_t K, float sigma, uint32_t T,
                        uint32_t m, float eta, uint32_t iters, float* loss, void* stream) {
  int rc = check_kparams(npix, K, sigma, T, m);
  if (rc) return rc;
  if (!std::isfinite(eta) || eta <= 0.f) return fail(SRT3D_EINVAL, "eta=%g must be finite and > 0", (double)eta);
  if (iters > (1u << 24)) return fail(SRT3D_EINVAL, "iters=%u too large", iters);
  if (npix == 0 || (iters == 0 && !loss)) return SRT3D_OK;
  if (!z || !t || !alpha) return fail(SRT3D_ENULL, "z/t/alpha must be non-NULL");
  if (!aligned(z, 8) || !aligned(t, 4) || !aligned(alpha, 4) || (loss && !aligned(loss, 4)))
    return fail(SRT3D_EALIGN, "z must be 8-byte and t/alpha/loss 4-byte aligned");
  srt3d::PixArgs a = {};
  fill_consts(a, sigma, T, m, eta);
  a.z = z;
  a.t_in = t;
  a.a_in = alpha;
  a.t_out = t;
  a.a_out = alpha;
  a.loss = loss;
  a.npix = npix;
  cudaError_t e = srt3d::launch_fit((int)K, a, (int)iters, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_fit_pixelwise");
  return SRT3D_OK;
}

// ---- NEXT-3 initialisation ---------------------------------------------------
static int init_args(srt3d::BpArgs& b, const float* z, int64_t npix, float sigma, uint32_t T, uint32_t m) {
  int rc = check_kparams(npix, 1, sigma, T, m);
  if (rc) return rc;
  srt3d::PixArgs pa = {};
  fill_consts(pa, sigma, T, m, 1.f);
  double sh2 = 0.0;
  for (uint32_t j = 1; j <= m; j++) {
    const double w = 2.0 * 3.14159265358979323846 * (double)j / (double)T;
    const double h = std::exp(-(double)sigma * (double)sigma * w * w / 2.0);
    sh2 += h * h;
  }
  b = {};
  for (int j = 0; j < srt3d::MAX_M; j++) b.hh[j] = pa.c.hh[j];
  b.inv_sh2 = (float)(1.0 / sh2);
  b.z = z;
  b.npix = npix;
  b.T = T;
  b.m = m;
  return SRT3D_OK;
}

int srt3d_backproject(const float* z, int64_t npix, float sigma, uint32_t T, uint32_t m, uint32_t N, float* g,
                      void* stream) {
  srt3d::BpArgs b;
  int rc = init_args(b, z, npix, sigma, T, m);
  if (rc) return rc;
  if (N < 1 || N > 8192) return fail(SRT3D_EINVAL, "N=%u must be in [1, 8192]", N);
  if (npix == 0) return SRT3D_OK;
  if (!z || !g) return fail(SRT3D_ENULL, "z/g must be non-NULL");
  if (!aligned(z, 8) || !aligned(g, 4)) return fail(SRT3D_EALIGN, "z must be 8-byte and g 4-byte aligned");
  b.g = g;
  b.N = N;
  cudaError_t e = srt3d::launch_backproject(b, false, (cudaStream_t)stream, num_sms_current());
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_backproject");
  return SRT3D_OK;
}

int srt3d_init_depths(const float* z, int64_t npix, float sigma, uint32_t T, uint32_t m, uint32_t N, uint32_t K,
                      uint32_t min_sep, float* t, float* g_at, float* alpha, int32_t* count, void* stream) {
  srt3d::BpArgs b;
  int rc = init_args(b, z, npix, sigma, T, m);
  if (rc) return rc;
  if (N < 3 || N > 4096) return fail(SRT3D_EINVAL, "N=%u must be in [3, 4096]", N);
  if (K < 1) return fail(SRT3D_EINVAL, "K=%u < 1", K);
  if (K > SRT3D_MAX_K) return fail(SRT3D_EUNSUPPORTED, "K=%u exceeds SRT3D_MAX_K=%u", K, SRT3D_MAX_K);
  if (npix == 0) return SRT3D_OK;
  if (!z || !t || !g_at || !alpha || !count) return fail(SRT3D_ENULL, "z/t/g_at/alpha/count must be non-NULL");
  if (!aligned(z, 8) || !aligned(t, 4) || !aligned(g_at, 4) || !aligned(alpha, 4) || !aligned(count, 4))
    return fail(SRT3D_EALIGN, "z must be 8-byte and the outputs 4-byte aligned");
  b.N = N;
  b.K = K;
  b.min_sep = min_sep;
  b.t_out = t;
  b.g_out = g_at;
  b.a_out = alpha;
  b.count = count;
  cudaError_t e = srt3d::launch_backproject(b, true, (cudaStream_t)stream, num_sms_current());
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_init_depths");
  return SRT3D_OK;
}

int srt3d_init_k1(const float* z, int64_t npix, float sigma, uint32_t T, uint32_t m, float* t, float* alpha,
                  void* stream) {
  srt3d::BpArgs b;
  int rc = init_args(b, z, npix, sigma, T, m);
  if (rc) return rc;
  if (npix == 0) return SRT3D_OK;
  if (!z || !t || !alpha) return fail(SRT3D_ENULL, "z/t/alpha must be non-NULL");
  if (!aligned(z, 8) || !aligned(t, 4) || !aligned(alpha, 4))
    return fail(SRT3D_EALIGN, "z must be 8-byte and t/alpha 4-byte aligned");
  b.t_out = t;
  b.a_out = alpha;
  cudaError_t e = srt3d::launch_init_k1(b, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_init_k1");
  return SRT3D_OK;
}

// ---- NEXT-4 streaming acquisition -------------------------------------------
int srt3d_sketch_merge(const float* za, const uint32_t* na, const float* zb, const uint32_t* nb, int64_t npix,
                       uint32_t m, float* z_out, uint32_t* n_out, void* stream) {
  if (npix < 0) return fail(SRT3D_EINVAL, "npix=%lld < 0", (long long)npix);
  if (m < 1) return fail(SRT3D_EINVAL, "m=%u < 1", m);
  if (m > SRT3D_MAX_M) return fail(SRT3D_EUNSUPPORTED, "m=%u exceeds SRT3D_MAX_M=%u", m, SRT3D_MAX_M);
  if (npix == 0) return SRT3D_OK;
  if (!za || !na || !zb || !nb || !z_out || !n_out) return fail(SRT3D_ENULL, "all pointers must be non-NULL");
  if (!aligned(za, 8) || !aligned(zb, 8) || !aligned(z_out, 8) || !aligned(na, 4) || !aligned(nb, 4) ||
      !aligned(n_out, 4))
    return fail(SRT3D_EALIGN, "z must be 8-byte and n 4-byte aligned");
  cudaError_t e = srt3d::launch_merge(za, na, zb, nb, nullptr, npix, m, z_out, n_out, (cudaStream_t)stream,
                                      num_sms_current());
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_sketch_merge");
  return SRT3D_OK;
}

int srt3d_sketch_accumulate(float* z, uint32_t* n, const float* zb, const uint32_t* offsets_b, int64_t npix,
                            uint32_t m, void* stream) {
  if (npix < 0) return fail(SRT3D_EINVAL, "npix=%lld < 0", (long long)npix);
  if (m < 1) return fail(SRT3D_EINVAL, "m=%u < 1", m);
  if (m > SRT3D_MAX_M) return fail(SRT3D_EUNSUPPORTED, "m=%u exceeds SRT3D_MAX_M=%u", m, SRT3D_MAX_M);
  if (npix == 0) return SRT3D_OK;
  if (!z || !n || !zb || !offsets_b) return fail(SRT3D_ENULL, "all pointers must be non-NULL");
  if (!aligned(z, 8) || !aligned(zb, 8) || !aligned(n, 4) || !aligned(offsets_b, 4))
    return fail(SRT3D_EALIGN, "z must be 8-byte and n/offsets 4-byte aligned");
  cudaError_t e = srt3d::launch_merge(z, n, zb, nullptr, offsets_b, npix, m, z, n, (cudaStream_t)stream,
                                      num_sms_current());
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_sketch_accumulate");
  return SRT3D_OK;
}

uint64_t srt3d_bucket_scratch_words(int64_t npix, uint64_t nevents) {
  return npix < 0 ? 0 : (uint64_t)srt3d::bucket_scratch_words(npix, nevents);
}

int srt3d_bucket_events(const uint32_t* pix, const uint16_t* bins, uint64_t nevents, int64_t npix,
                        uint32_t* offsets, uint16_t* bins_out, uint32_t* scratch, uint32_t* dropped, void* stream) {
  if (npix < 0) return fail(SRT3D_EINVAL, "npix=%lld < 0", (long long)npix);
  if (nevents >= (1ull << 32)) return fail(SRT3D_EINVAL, "nevents=%llu must be < 2^32", (unsigned long long)nevents);
  if (!offsets || !scratch) return fail(SRT3D_ENULL, "offsets/scratch must be non-NULL");
  if (nevents && (!pix || !bins || !bins_out)) return fail(SRT3D_ENULL, "pix/bins/bins_out must be non-NULL");
  if (!aligned(pix, 4) || !aligned(bins, 2) || !aligned(offsets, 4) || !aligned(bins_out, 2) ||
      !aligned(scratch, 4) || (dropped && !aligned(dropped, 4)))
    return fail(SRT3D_EALIGN, "pix/offsets/scratch/dropped 4-byte and bins 2-byte aligned");
  cudaError_t e = srt3d::launch_bucket(pix, bins, nevents, npix, offsets, bins_out, scratch, dropped,
                                       (cudaStream_t)stream, num_sms_current());
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_bucket_events");
  return SRT3D_OK;
}

int srt3d_check_csr(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, int32_t* bad,
                    void* stream) {
  if (npix < 0) return fail(SRT3D_EINVAL, "npix=%lld < 0", (long long)npix);
  if (T < 2 || T > SRT3D_MAX_T) return fail(SRT3D_EINVAL, "T=%u out of range", T);
  if (npix == 0) return SRT3D_OK;
  if (!bins || !offsets || !bad) return fail(SRT3D_ENULL, "bins/offsets/bad must be non-NULL");
  cudaError_t e = srt3d::launch_check_csr(bins, offsets, npix, T, bad, (cudaStream_t)stream, num_sms_current());
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_check_csr");
  return SRT3D_OK;
}

int srt3d_debug_ffma_peak(double* tflops) {
  if (!tflops) return fail(SRT3D_ENULL, "tflops must be non-NULL");
  cudaError_t e = srt3d::measure_ffma_peak(tflops, num_sms_current());
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_debug_ffma_peak");
  return SRT3D_OK;
}

int srt3d_debug_phase_index(const uint16_t* bins, int64_t n, uint32_t T, uint32_t m, uint32_t* r, void* stream) {
  if (n < 0) return fail(SRT3D_EINVAL, "n=%lld < 0", (long long)n);
  if (T < 2 || T > SRT3D_MAX_T) return fail(SRT3D_EINVAL, "T=%u out of range", T);
  if (m < 1 || m > SRT3D_MAX_M) return fail(SRT3D_EINVAL, "m=%u out of range", m);
  if (n == 0) return SRT3D_OK;
  if (!bins || !r) return fail(SRT3D_ENULL, "bins/r must be non-NULL");
  if (!aligned(r, 4)) return fail(SRT3D_EALIGN, "r must be 4-byte aligned");
  cudaError_t e = srt3d::launch_phase_index(bins, n, T, m, r, (cudaStream_t)stream, num_sms_current());
  if (e != cudaSuccess) return cuda_fail(e, "srt3d_debug_phase_index");
  return SRT3D_OK;
}

}  // extern "C"
