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

int num_sms_current() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

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

int lanes_for(double mean_photons) {
  // >= ~100 photons per lane amortises the group reduce-scatter and the
  // head/tail peel (tools/sketch_tune.cu: G=8 beats G=16 at n=1000, m=32)
  if (mean_photons >= 4096.0) return 32;
  if (mean_photons >= 2048.0) return 16;
  if (mean_photons >= 256.0) return 8;
  return 4;
}

bool pair_fits(uint32_t T) { return T <= srt3d::SO_MAX_T; }

int choose_path(uint32_t T, uint32_t m, double mean, int* lanes) {
  const int M0 = (int)(m < 32 ? m : 32);
  const bool hist_fits = srt3d::sketch_hist_smem(T, M0) <= 227u * 1024u;
  int path = SRT3D_PATH_DIRECT;
  if (hist_fits && mean >= SRT3D_BINCOUNT_MIN_PHOTONS_PER_BIN * (double)T) path = SRT3D_PATH_BINCOUNT;
  int G = lanes_for(mean);
  if (G == 8 && M0 >= 24) G = 4;  // the G = 4 rotated-Chebyshev regime of srt3d_sketch_ex
  if (lanes) *lanes = path == SRT3D_PATH_BINCOUNT ? 0 : (path == SRT3D_PATH_PAIRED ? 32 : G);
  return path;
}

}  // namespace

extern "C" {

int srt3d_version(void) { return 100; }

const char* srt3d_last_error(void) { return g_err; }

int srt3d_sketch_ex(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, uint32_t m, float* z,
                    uint64_t total_photons_hint, int path, int lanes_per_pixel, void* stream) {
  if (npix < 0) return fail(SRT3D_EINVAL, "npix=%lld < 0", (long long)npix);
  int rc = check_tm(T, m);
  if (rc) return rc;
  if (path < SRT3D_PATH_AUTO || path > SRT3D_PATH_PAIRED) return fail(SRT3D_EINVAL, "path=%d unknown", path);
  if (lanes_per_pixel != 0 && lanes_per_pixel != 4 && lanes_per_pixel != 8 && lanes_per_pixel != 16 &&
      lanes_per_pixel != 32)
    return fail(SRT3D_EINVAL, "lanes_per_pixel=%d must be 0, 4, 8, 16 or 32", lanes_per_pixel);
  if (npix == 0) return SRT3D_OK;
  if (!offsets || !z) return fail(SRT3D_ENULL, "offsets/z must be non-NULL");
  if (!bins && total_photons_hint != 0) return fail(SRT3D_ENULL, "bins must be non-NULL");
  if (!aligned(bins, 2) || !aligned(offsets, 4) || !aligned(z, 8))
    return fail(SRT3D_EALIGN, "bins/offsets/z must be 2/4/8-byte aligned");
  const int M0 = (int)(m < 32 ? m : 32);
  const bool hist_fits = srt3d::sketch_hist_smem(T, M0) <= 227u * 1024u;
  if (path == SRT3D_PATH_BINCOUNT && !hist_fits)
    return fail(SRT3D_EUNSUPPORTED, "bin-count path needs T <= ~17000 (T=%u)", T);
  if (path == SRT3D_PATH_PAIRED && !pair_fits(T))
    return fail(SRT3D_EUNSUPPORTED, "class-sorted path needs T <= %u (T=%u)", srt3d::SO_MAX_T, T);
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t total = total_photons_hint;
  if (total == 0 && (path == SRT3D_PATH_AUTO || lanes_per_pixel == 0)) {
    uint32_t ends[2] = {0, 0};
    cudaError_t e = cudaMemcpyAsync(&ends[0], offsets, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&ends[1], offsets + npix, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "srt3d_sketch(read offsets)");
    total = ends[1] >= ends[0] ? (uint64_t)(ends[1] - ends[0]) : 0;
  }
  if (!bins && total != 0) return fail(SRT3D_ENULL, "bins must be non-NULL");
  const double mean = (double)total / (double)npix;
  if (path == SRT3D_PATH_AUTO) path = choose_path(T, m, mean, nullptr);
  const int G = lanes_per_pixel ? lanes_per_pixel : lanes_for(mean);
  const int nsm = num_sms_current();
  srt3d::SketchArgs a;
  a.bins = bins ? bins : reinterpret_cast<const uint16_t*>(offsets);  // never dereferenced when no photons
  a.offsets = offsets;
  a.npix = npix;
  a.T = T;
  a.mstride = m;
  a.z = z;
  for (uint32_t j0 = 0; j0 < m; j0 += 32) {
    a.j0 = j0;
    const int M = (int)((m - j0) < 32 ? (m - j0) : 32);
    // auto regime, long passes at ~1e3 photons/pixel: G = 4 + rotated
    // Chebyshev beats G = 8 + complex power
    const int Gp = (lanes_per_pixel == 0 && G == 8 && M >= 24) ? srt3d::SK_G4_CHEB : G;
    cudaError_t e = path == SRT3D_PATH_BINCOUNT ? srt3d::launch_sketch_hist(M, a, mean, s, nsm)
                    : path == SRT3D_PATH_PAIRED ? srt3d::launch_sketch_pair(M, a, s, nsm)
                                                : srt3d::launch_sketch_pass(M, Gp, a, s, nsm);
    if (e != cudaSuccess) return cuda_fail(e, "srt3d_sketch");
  }
  return SRT3D_OK;
}

int srt3d_sketch_plan(int64_t npix, uint32_t T, uint32_t m, uint64_t total_photons, int* lanes_per_pixel) {
  if (npix <= 0) return fail(SRT3D_EINVAL, "npix=%lld must be > 0", (long long)npix);
  int rc = check_tm(T, m);
  if (rc) return rc;
  return choose_path(T, m, (double)total_photons / (double)npix, lanes_per_pixel);
}

int srt3d_sketch(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, uint32_t m, float* z,
                 uint64_t total_photons_hint, void* stream) {
  return srt3d_sketch_ex(bins, offsets, npix, T, m, z, total_photons_hint, SRT3D_PATH_AUTO, 0, stream);
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
