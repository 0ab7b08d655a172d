// K2 / K3 / K4 — per-pixel model sketch, sketched loss + gradient, update.
//
//   Phi_j   = sum_k alpha_k hhat_j exp(i omega_j t_k)            Eq. (4)
//   r_j     = z_j - Phi_j ;  L = sum_j |r_j|^2                  Eq. (6)/(8), W = I
//   dL/dalpha_k = -2 sum_j hhat_j Re(conj r_j e^{i omega_j t_k})
//   dL/dt_k     = +2 alpha_k sum_j omega_j hhat_j Im(conj r_j e^{i omega_j t_k})
//
// One thread per pixel, looping over j = 1..m with the K phasors
// p_jk = exp(i omega_j t_k) advanced by the packed complex recurrence
// p_jk = p_{j-1,k} * w_k.  The base w_k comes from an exact 32-bit
// fixed-point phase q_k = round(frac(t_k / T) 2^32) (so j*t_k needs no fp32
// range reduction), re-anchored every 32 frequencies from j*q_k; worst-case
// phasor error 1.6e-6 (tools/sim_grad_phasor_error.py).
// Per (j, k): 2 (phasor) + 1 (Phi) + 2 (gradient) packed FP32x2 instructions.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace srt3d {

template <int M>
struct ConstView {
  const float* hh;
  const float* wh;
};

template <int K, int M, int MODE>
__global__ void __launch_bounds__(PX_THREADS) pixel_kernel(const PixArgs a) {
  // Frequency constants: compile-time-indexed kernel parameters when M is a
  // template constant; staged in shared memory for the runtime-m variant.
  __shared__ float s_hh[M == 0 ? MAX_M : 1], s_wh[M == 0 ? MAX_M : 1];
  if (M == 0 && MODE != PX_UPDATE) {
    for (int j = threadIdx.x; j < MAX_M; j += blockDim.x) {
      s_hh[j] = a.c.hh[j];
      s_wh[j] = a.c.wh[j];
    }
    __syncthreads();
  }
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npix) return;
  const int m = M ? M : (int)a.m;

  float tk[K], ak[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    tk[k] = a.t_in[i * K + k];
    ak[k] = a.a_in[i * K + k];
  }

  if (MODE == PX_UPDATE) {
#pragma unroll
    for (int k = 0; k < K; k++) {
      const float gt = a.grad_t[i * K + k], ga = a.grad_a[i * K + k];
      const float am = fmaxf(ak[k], 0.05f);
      float step = a.eta * gt * a.upd_t_scale / (am * am);
      step = fminf(fmaxf(step, -a.max_step), a.max_step);
      float tn = tk[k] - step;
      tn = tn - a.Tf * floorf(tn / a.Tf);
      if (tn >= a.Tf) tn -= a.Tf;
      if (tn < 0.f) tn += a.Tf;
      a.t_out[i * K + k] = tn;
      a.a_out[i * K + k] = fminf(fmaxf(ak[k] - a.eta * ga * a.upd_a_scale, 0.f), 1.f);
    }
    return;
  }

  uint32_t q[K];
  u64 W[K], Wn[K], P[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    q[k] = phase_q32(tk[k], a.invT);
    const float2 w = phasor_q32(q[k]);
    W[k] = pk(w.x, w.y);
    Wn[k] = pk(-w.y, w.x);
    P[k] = W[k];
  }

  float L = 0.f;
  u64 GA[K], GT[K];  // packed partial sums: GA = sum (rho_r p_r, rho_i p_i); GT = sum (s_r p_i, -s_i p_r)
#pragma unroll
  for (int k = 0; k < K; k++) {
    GA[k] = 0ull;
    GT[k] = 0ull;
  }
  const float2* zrow = reinterpret_cast<const float2*>(a.z) + (size_t)i * m;
  float2* zout = reinterpret_cast<float2*>(a.zout) + (size_t)i * m;

#pragma unroll(M ? M : 1)
  for (int j = 0; j < m; j++) {  // frequency j+1
    if (j > 0) {
      if ((j & 31) == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) {
          const float2 p = phasor_q32(q[k] * (uint32_t)(j + 1));
          P[k] = pk(p.x, p.y);
        }
      } else {
#pragma unroll
        for (int k = 0; k < K; k++) P[k] = cmul2(P[k], W[k], Wn[k]);
      }
    }
    const float hh = M ? a.c.hh[j] : s_hh[j];
    // S = sum_k alpha_k p_jk  (Phi_j = hh * S)
    u64 S = fmul2(pk(ak[0], ak[0]), P[0]);
#pragma unroll
    for (int k = 1; k < K; k++) S = ffma2(pk(ak[k], ak[k]), P[k], S);
    if (MODE == PX_EXPECTED) {
      zout[j] = make_float2(hh * lo_of(S), hh * hi_of(S));
      continue;
    }
    const float wh = M ? a.c.wh[j] : s_wh[j];
    const float2 zj = __ldg(zrow + j);
    const float rr = fmaf(-hh, lo_of(S), zj.x);
    const float ri = fmaf(-hh, hi_of(S), zj.y);
    L = fmaf(rr, rr, fmaf(ri, ri, L));
    const u64 RHO = pk(hh * rr, hh * ri);   // hhat_j r_j
    const u64 SIG = pk(wh * rr, -wh * ri);  // omega_j hhat_j (r_r, -r_i)
#pragma unroll
    for (int k = 0; k < K; k++) {
      GA[k] = ffma2(RHO, P[k], GA[k]);                             // (rho_r p_r, rho_i p_i)
      GT[k] = ffma2(SIG, pk(hi_of(P[k]), lo_of(P[k])), GT[k]);     // (s_r p_i, -s_i p_r)
    }
  }
  if (MODE == PX_EXPECTED) return;

  float gt[K], ga[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    ga[k] = -2.f * (lo_of(GA[k]) + hi_of(GA[k]));
    gt[k] = 2.f * ak[k] * (lo_of(GT[k]) + hi_of(GT[k]));
  }
  if (a.loss) a.loss[i] = L;
  if (MODE == PX_GRAD) {
#pragma unroll
    for (int k = 0; k < K; k++) {
      a.grad_t[i * K + k] = gt[k];
      a.grad_a[i * K + k] = ga[k];
    }
    return;
  }
  // PX_GRAD_STEP: fused update (same arithmetic as PX_UPDATE)
#pragma unroll
  for (int k = 0; k < K; k++) {
    const float am = fmaxf(ak[k], 0.05f);
    float step = a.eta * gt[k] * a.upd_t_scale / (am * am);
    step = fminf(fmaxf(step, -a.max_step), a.max_step);
    float tn = tk[k] - step;
    tn = tn - a.Tf * floorf(tn / a.Tf);
    if (tn >= a.Tf) tn -= a.Tf;
    if (tn < 0.f) tn += a.Tf;
    a.t_out[i * K + k] = tn;
    a.a_out[i * K + k] = fminf(fmaxf(ak[k] - a.eta * ga[k] * a.upd_a_scale, 0.f), 1.f);
  }
}

template <int K, int M, int MODE>
static cudaError_t launch_px(const PixArgs& a, cudaStream_t s) {
  const long long grid = (a.npix + PX_THREADS - 1) / PX_THREADS;
  pixel_kernel<K, M, MODE><<<(unsigned)grid, PX_THREADS, 0, s>>>(a);
  return cudaGetLastError();
}

template <int K, int MODE>
static cudaError_t launch_px_m(const PixArgs& a, cudaStream_t s) {
  if (MODE == PX_UPDATE) return launch_px<K, 0, MODE>(a, s);
  if (K <= 3) {
    switch (a.m) {
      case 4:
        return launch_px<K, 4, MODE>(a, s);
      case 5:
        return launch_px<K, 5, MODE>(a, s);
      case 10:
        return launch_px<K, 10, MODE>(a, s);
      case 20:
        return launch_px<K, 20, MODE>(a, s);
      case 32:
        return launch_px<K, 32, MODE>(a, s);
      default:
        break;
    }
  }
  return launch_px<K, 0, MODE>(a, s);
}

template <int MODE>
static cudaError_t launch_px_k(int K, const PixArgs& a, cudaStream_t s) {
  switch (K) {
    case 1:
      return launch_px_m<1, MODE>(a, s);
    case 2:
      return launch_px_m<2, MODE>(a, s);
    case 3:
      return launch_px_m<3, MODE>(a, s);
    case 4:
      return launch_px_m<4, MODE>(a, s);
    case 5:
      return launch_px_m<5, MODE>(a, s);
    case 6:
      return launch_px_m<6, MODE>(a, s);
    case 7:
      return launch_px_m<7, MODE>(a, s);
    case 8:
      return launch_px_m<8, MODE>(a, s);
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pixel(PixMode mode, int K, const PixArgs& a, cudaStream_t s) {
  if (a.npix <= 0) return cudaSuccess;
  switch (mode) {
    case PX_EXPECTED:
      return launch_px_k<PX_EXPECTED>(K, a, s);
    case PX_GRAD:
      return launch_px_k<PX_GRAD>(K, a, s);
    case PX_GRAD_STEP:
      return launch_px_k<PX_GRAD_STEP>(K, a, s);
    case PX_UPDATE:
      return launch_px_k<PX_UPDATE>(K, a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace srt3d
