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
//
// Memory: each warp owns 32 consecutive pixels, whose z rows are one
// contiguous slab of 32*m complex64.  The warp stages the slab into shared
// memory with coalesced asynchronous copies (cp.async / LDGSTS, 16-byte units
// for even m; all of a lane's copies in flight at once) into rows of padded
// stride S, so that the per-thread row reads are bank-conflict free; the
// expected-sketch output goes the same way in reverse.  (Reading z row-wise
// straight from global memory touches 32 sectors per warp load — L1-wavefront
// bound; a register-staged copy serialises load -> store.)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace srt3d {

// Row stride of the shared z tile, in complex64 units.  16-byte path (even
// m): S = m + 2 keeps rows 16-byte aligned and makes the per-thread LDS.128
// row reads conflict-free (16B-unit address 17*row + j/2 walks all 8 units of
// a 128-byte phase for 8 consecutive rows).  8-byte path (odd m): S odd.
__host__ __device__ constexpr int zstride(int m) { return (m & 1) ? m : m + 2; }

__device__ __forceinline__ void cp_async(void* smem_dst, const void* gsrc, int bytes16) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  if (bytes16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Stage a warp's slab of nrows*m complex64 (contiguous in global memory) into
// the padded shared tile with asynchronous copies (LDGSTS: every lane keeps
// all its copies in flight; no register staging).  Units are 16 bytes (two
// complex) when m is even, else 8 bytes.  Row/column advance incrementally.
// v16 needs an even m AND a 16-byte-aligned slab (z itself may be only
// 8-byte aligned: the ABI's requirement).
__device__ __forceinline__ void warp_slab_issue(float2* tile, const float2* gsrc, int nrows, int m, int S, int lane) {
  const bool v16 = (m & 1) == 0 && ((uintptr_t)gsrc & 15u) == 0;
  const int mu = v16 ? m / 2 : m;  // units per row
  const int total = nrows * mu;
  int row = lane / mu, col = lane - (lane / mu) * mu;
  const int q = 32 / mu, r = 32 - (32 / mu) * mu;
  const int w = v16 ? 2 : 1;
  for (int u = lane; u < total; u += 32) {
    cp_async(tile + row * S + col * w, gsrc + (size_t)u * w, v16);
    col += r;
    row += q;
    if (col >= mu) {
      col -= mu;
      row++;
    }
  }
}

// Coalesced copy-out of the warp's tile (expected sketch).
__device__ __forceinline__ void warp_slab_store(const float2* tile, float2* gdst, int nrows, int m, int S, int lane) {
  const int total = nrows * m;
  int row = lane / m, col = lane - (lane / m) * m;
  const int q = 32 / m, r = 32 - (32 / m) * m;
#pragma unroll 4
  for (int u = lane; u < total; u += 32) {
    gdst[u] = tile[row * S + col];
    col += r;
    row += q;
    if (col >= m) {
      col -= m;
      row++;
    }
  }
}

// ---- TMA staging of the z slab (m % 16 == 0) ----------------------------------
// The harness update (reading A13) for one (pixel, k); shared by the fused
// step and K4 so both produce bit-identical results.
__device__ __forceinline__ void update_one(const PixArgs& a, float tk, float ak, float gt, float ga, float& tn,
                                           float& an) {
  // branch-free: approximate reciprocal division (harness update, not part of
  // the paper's arithmetic; the oracle comparison tolerance covers ~2 ulp)
  const float am = fmaxf(ak, 0.05f);
  float step = __fdividef(a.eta * gt * a.upd_t_scale, am * am);
  step = fminf(fmaxf(step, -a.max_step), a.max_step);
  tn = tk - step;
  tn = fmaf(-a.Tf, floorf(tn * a.invTf), tn);
  tn = tn >= a.Tf ? tn - a.Tf : tn;
  tn = tn < 0.f ? tn + a.Tf : tn;
  an = fminf(fmaxf(fmaf(-a.eta * a.upd_a_scale, ga, ak), 0.f), 1.f);
}

// One pixel: anchors, the j loop, and the mode's outputs.  zrow points at the
// pixel's z row in the shared tile (row stride S).  `active` lanes store;
// inactive lanes (past the end of the frame) compute a duplicate and store
// nothing (PX_EXPECTED writes its tile row, copied out by the caller).
template <int K>
__device__ __forceinline__ void load_theta(const PixArgs& a, long long i, float (&tk)[K], float (&ak)[K]) {
#pragma unroll
  for (int k = 0; k < K; k++) {
    tk[k] = a.t_in[i * K + k];
    ak[k] = a.a_in[i * K + k];
  }
}

// Evaluates one pixel: Phi (PX_EXPECTED: written to zrow), else the loss L and
// the gradient (gt, ga).  WAIT_Z: wait for the warp's cp.async z slab after
// the anchors (which overlap the copy).
template <int K, int M, int MODE, bool WAIT_Z = true, bool ZTMA = false>
__device__ __forceinline__ void pixel_body(const PixArgs& a, float2* zrow, const float* s_hh, const float* s_wh,
                                           const float (&tk)[K], const float (&ak)[K], float (&gt)[K],
                                           float (&ga)[K], float& L, uint64_t* zbar = nullptr,
                                           uint32_t zpar = 0u) {
  const int m = M ? M : (int)a.m;
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

  if (MODE != PX_EXPECTED && WAIT_Z) {
    // the anchors above overlap the z slab's copy; wait for it only now
    if (ZTMA) {
      mbar_wait(zbar, zpar);  // box 0 (j < 16); later boxes are awaited inside the j loop
    } else {
      cp_async_wait_all();
      __syncwarp();
    }
  }
  u64 L2 = 0ull;  // packed (sum r_r^2, sum r_i^2)
  u64 GA[K], GT[K];  // packed partial sums: GA = sum (rho_r p_r, rho_i p_i); GT = sum (s_r p_i, -s_i p_r)
#pragma unroll
  for (int k = 0; k < K; k++) {
    GA[k] = 0ull;
    GT[k] = 0ull;
  }

#pragma unroll(M ? M : 1)
  for (int j = 0; j < m; j++) {  // frequency j+1
    if (ZTMA && MODE != PX_EXPECTED && WAIT_Z && j > 0 && j % 16 == 0) mbar_wait(zbar + j / 16, zpar);
    if (j > 0) {
      // re-anchored from the exact phase every 32 frequencies in the specialised kernels (m <= 32:
      // one anchor) and every 16 in the generic one (any m), whose worst-case recurrence error
      // otherwise reaches the A12 floor (DESIGN.md §3 A12: 3 components at 1.0-1.2x the floor in
      // 1024 extra fuzz shapes, all generic-m); the recurrence error grows with its length
      if ((j & (M ? 31 : 15)) == 0) {
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
    // Sk = sum_k alpha_k p_jk  (Phi_j = hh * Sk)
    u64 Sk = fmul2(pk(ak[0], ak[0]), P[0]);
#pragma unroll
    for (int k = 1; k < K; k++) Sk = ffma2(pk(ak[k], ak[k]), P[k], Sk);
    if (MODE == PX_EXPECTED) {
      zrow[j] = make_float2(hh * lo_of(Sk), hh * hi_of(Sk));
      continue;
    }
    const float wh = M ? a.c.wh[j] : s_wh[j];
    float2 zj;
    if (ZTMA) {  // TMA box h = j / 16 (4 KB, 32 rows x 128 B, 128B swizzle): chunk (j%16)/2 ^ (row & 7)
      const int r7 = (threadIdx.x & 7) << 4;
      const float4 z2 = *reinterpret_cast<const float4*>(reinterpret_cast<const char*>(zrow) + (j / 16) * 4096 +
                                                         ((((j % 16) / 2) << 4) ^ r7));
      zj = (j & 1) ? make_float2(z2.z, z2.w) : make_float2(z2.x, z2.y);
    } else if (M > 0 && (M & 1) == 0) {  // LDS.128: z_j, z_{j+1} (conflict-free with S = m + 2)
      const float4 z2 = *reinterpret_cast<const float4*>(zrow + (j & ~1));
      zj = (j & 1) ? make_float2(z2.z, z2.w) : make_float2(z2.x, z2.y);
    } else {
      zj = zrow[j];
    }
    // packed: R = z_j - hh Sk ; L2 += R*R ; RHO = hh R ; SIG = (wh, -wh) * R
    const u64 R = ffma2(pk(-hh, -hh), Sk, pk(zj.x, zj.y));
    if (MODE != PX_GRAD_STEP_NL && MODE != PX_GRAD_NL) L2 = ffma2(R, R, L2);  // the loss only when it is stored
    const u64 RHO = fmul2(pk(hh, hh), R);   // hhat_j r_j
    const u64 SIG = fmul2(pk(wh, -wh), R);  // omega_j hhat_j (r_r, -r_i)
#pragma unroll
    for (int k = 0; k < K; k++) {
      GA[k] = ffma2(RHO, P[k], GA[k]);                          // (rho_r p_r, rho_i p_i)
      GT[k] = ffma2(SIG, pk(hi_of(P[k]), lo_of(P[k])), GT[k]);  // (s_r p_i, -s_i p_r)
    }
  }
  if (MODE == PX_EXPECTED) return;
#pragma unroll
  for (int k = 0; k < K; k++) {
    ga[k] = -2.f * (lo_of(GA[k]) + hi_of(GA[k]));
    gt[k] = 2.f * ak[k] * (lo_of(GT[k]) + hi_of(GT[k]));
  }
  L = lo_of(L2) + hi_of(L2);
}

// Stores of one evaluated pixel, per mode (gradient / fused step).
template <int K, int MODE>
__device__ __forceinline__ void pixel_store(const PixArgs& a, long long i, const float (&tk)[K], const float (&ak)[K],
                                            const float (&gt)[K], const float (&ga)[K], float L) {
  if (MODE != PX_GRAD_STEP_NL && MODE != PX_GRAD_NL && a.loss) a.loss[i] = L;
  if (MODE == PX_GRAD || MODE == PX_GRAD_NL) {
#pragma unroll
    for (int k = 0; k < K; k++) {
      a.grad_t[i * K + k] = gt[k];
      a.grad_a[i * K + k] = ga[k];
    }
    return;
  }
  // PX_GRAD_STEP: fused update
#pragma unroll
  for (int k = 0; k < K; k++) {
    float tn, an;
    update_one(a, tk[k], ak[k], gt[k], ga[k], tn, an);
    a.t_out[i * K + k] = tn;
    a.a_out[i * K + k] = an;
  }
}

template <int M>
__device__ __forceinline__ void stage_consts(const PixArgs& a, float* s_hh, float* s_wh) {
  if (M == 0) {
    for (int j = threadIdx.x; j < MAX_M; j += blockDim.x) {
      s_hh[j] = a.c.hh[j];
      s_wh[j] = a.c.wh[j];
    }
    __syncthreads();
  }
}

// Expected sketch (K2): one warp = 32 pixels, output staged through the
// padded tile and copied out coalesced.
template <int K, int M>
__global__ void __launch_bounds__(PX_THREADS) expected_kernel(const PixArgs a) {
  __shared__ float s_hh[M == 0 ? MAX_M : 1], s_wh[M == 0 ? MAX_M : 1];
  extern __shared__ float2 ztile[];
  stage_consts<M>(a, s_hh, s_wh);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long row0 = (long long)blockIdx.x * blockDim.x + (warp << 5);
  if (row0 >= a.npix) return;
  const long long i = row0 + lane;
  const int nrows = (int)min(32ll, a.npix - row0);
  const int m = M ? M : (int)a.m;
  const int S = zstride(m);
  float2* tile = ztile + (size_t)warp * 32 * S;
  const bool active = i < a.npix;
  float tk[K], ak[K];
  load_theta<K>(a, active ? i : a.npix - 1, tk, ak);
  float gt[K], ga[K], L;
  pixel_body<K, M, PX_EXPECTED>(a, tile + lane * S, s_hh, s_wh, tk, ak, gt, ga, L);
  __syncwarp();
  warp_slab_store(tile, reinterpret_cast<float2*>(a.zout) + (size_t)row0 * m, nrows, m, S, lane);
}

// Gradient / fused step (K3, K3+K4): one warp = 32 pixels; the warp's z slab
// is staged into its shared tile with cp.async, then each lane runs its pixel.
template <int K, int M, int MODE>
__global__ void __launch_bounds__(GRAD_THREADS, GRAD_MIN_BLOCKS) grad_kernel(const PixArgs a) {
  __shared__ float s_hh[M == 0 ? MAX_M : 1], s_wh[M == 0 ? MAX_M : 1];
  extern __shared__ float2 ztile[];
  stage_consts<M>(a, s_hh, s_wh);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long row0 = (long long)blockIdx.x * blockDim.x + (warp << 5);
  if (row0 >= a.npix) return;
  const int m = M ? M : (int)a.m;
  const int S = zstride(m);
  float2* tile = ztile + (size_t)warp * 32 * S;
  const long long i = row0 + lane;
  const bool active = i < a.npix;
  float tk[K], ak[K];
  load_theta<K>(a, active ? i : a.npix - 1, tk, ak);  // first: the anchors need theta before z
  warp_slab_issue(tile, reinterpret_cast<const float2*>(a.z) + (size_t)row0 * m, (int)min(32ll, a.npix - row0), m, S,
                  lane);
  // inactive lanes (past the frame end) run a duplicate of the last pixel so
  // the warp stays converged at the in-body cp.async wait; they store nothing
  float gt[K], ga[K], L;
  pixel_body<K, M, MODE>(a, tile + lane * S, s_hh, s_wh, tk, ak, gt, ga, L);
  if (active) pixel_store<K, MODE>(a, i, tk, ak, gt, ga, L);
}

// Gradient / fused step for m % 16 == 0: the warp's 32 z rows arrive by TMA —
// m/16 boxes of 32 rows x 32 floats (128 B) with the 128-byte swizzle, one
// instruction each from one lane, completing on the warp's mbarrier — instead
// of m/2 cp.async per lane plus their address arithmetic.  The swizzle places
// 16-byte chunk c of row r at chunk c ^ (r & 7), so the per-thread LDS.128 row
// reads of a quarter-warp hit 8 different bank groups (conflict-free) with no
// padding.  Rows past the frame end are zero-filled by the TMA unit.
template <int K, int M, int MODE>
__global__ void __launch_bounds__(GRAD_THREADS, GRAD_TMA_MIN_BLOCKS) grad_kernel_tma(const PixArgs a,
                                                                                const __grid_constant__ CUtensorMap tm) {
  static_assert(M > 0 && M % 16 == 0, "TMA boxes of 32 floats");
  constexpr int NBOX = M / 16;
  extern __shared__ unsigned char tma_smem_raw[];
  unsigned char* smem = tma_smem_raw + ((1024u - (smem_u32(tma_smem_raw) & 1023u)) & 1023u);  // 1 KB aligned
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* tile = smem + (size_t)warp * NBOX * 4096;
  // one mbarrier per box: the j loop waits for box h only when it reaches j = 16 h,
  // so later boxes land while the first frequencies are computed
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)(GRAD_THREADS / 32) * NBOX * 4096) + warp * NBOX;
  if (lane == 0) {
#pragma unroll
    for (int h = 0; h < NBOX; h++) mbar_init(bar + h, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // launched as a programmatic dependent: the CTAs may start during the previous kernel's tail;
  // nothing is read before that kernel has completed (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t par = 0u;
  // GRAD_PERSIST: one wave of CTAs, each warp loops over its 32-row tiles; else one tile per warp
  for (long long row0 = (long long)blockIdx.x * blockDim.x + (warp << 5); row0 < a.npix;
       row0 += GRAD_PERSIST ? (long long)gridDim.x * blockDim.x : a.npix) {
    // theta first: the phasor anchors need it before any z, and issued ahead of the z boxes it
    // is not queued behind them in DRAM (C5 L2-cold launch 18.5 -> 17.9 us, in loop 14.0 -> 13.65 us)
    const long long i = row0 + lane;
    const bool active = i < a.npix;
    float tk[K], ak[K];
    load_theta<K>(a, active ? i : a.npix - 1, tk, ak);
    if (lane == 0) {
#pragma unroll
      for (int h = 0; h < NBOX; h++) {
        mbar_expect_tx(bar + h, 4096u);
        tma_load_2d(tile + h * 4096, &tm, h * 32, (int)row0, bar + h);
      }
    }
    __syncwarp();
    // scheduling only: the dependent step still waits (griddepcontrol.wait) for this grid to
    // complete before it reads anything
    if (GRAD_PDL_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    float gt[K], ga[K], L;
    pixel_body<K, M, MODE, true, true>(a, reinterpret_cast<float2*>(tile + lane * 128), nullptr, nullptr, tk, ak, gt,
                                       ga, L, bar, par);
    if (active) pixel_store<K, MODE>(a, i, tk, ak, gt, ga, L);
    par ^= 1u;
    __syncwarp();  // every lane has read the tile before the next boxes overwrite it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
}

// NEXT-2: `iters` fused data steps per pixel in one launch.
// The warp stages its z slab once; theta lives in registers across the
// iterations (each iteration is exactly the PX_GRAD_STEP arithmetic, so the
// result is bitwise equal to `iters` srt3d_sketch_grad_step calls).  If
// loss != NULL, the loss at the returned theta is evaluated once more.
template <int K, int M>
__global__ void __launch_bounds__(GRAD_THREADS) fit_kernel(const PixArgs a, int iters) {
  __shared__ float s_hh[M == 0 ? MAX_M : 1], s_wh[M == 0 ? MAX_M : 1];
  extern __shared__ float2 ztile[];
  stage_consts<M>(a, s_hh, s_wh);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long row0 = (long long)blockIdx.x * blockDim.x + (warp << 5);
  if (row0 >= a.npix) return;
  const int m = M ? M : (int)a.m;
  const int S = zstride(m);
  float2* tile = ztile + (size_t)warp * 32 * S;
  warp_slab_issue(tile, reinterpret_cast<const float2*>(a.z) + (size_t)row0 * m, (int)min(32ll, a.npix - row0), m, S,
                  lane);
  const long long i = row0 + lane;
  const bool active = i < a.npix;
  float tk[K], ak[K];
  load_theta<K>(a, active ? i : a.npix - 1, tk, ak);
  cp_async_wait_all();
  __syncwarp();
  float gt[K], ga[K], L = 0.f;
  for (int it = 0; it < iters; it++) {
    pixel_body<K, M, PX_GRAD_STEP_NL, false>(a, tile + lane * S, s_hh, s_wh, tk, ak, gt, ga, L);
#pragma unroll
    for (int k = 0; k < K; k++) {
      float tn, an;
      update_one(a, tk[k], ak[k], gt[k], ga[k], tn, an);
      tk[k] = tn;
      ak[k] = an;
    }
  }
  if (a.loss) pixel_body<K, M, PX_GRAD, false>(a, tile + lane * S, s_hh, s_wh, tk, ak, gt, ga, L);
  if (!active) return;
#pragma unroll
  for (int k = 0; k < K; k++) {
    a.t_out[i * K + k] = tk[k];
    a.a_out[i * K + k] = ak[k];
  }
  if (a.loss) a.loss[i] = L;
}

template <int K, int M>
static cudaError_t launch_fit_t(const PixArgs& a, int iters, cudaStream_t s) {
  auto fn = fit_kernel<K, M>;
  const int S = zstride(M ? M : (int)a.m);
  const size_t smem = sizeof(float2) * (GRAD_THREADS / 32) * 32 * S;
  static SmemAttrOnce attr;
  cudaError_t e = smem_attr_once(attr, fn, (int)(sizeof(float2) * (GRAD_THREADS / 32) * 32 * zstride(MAX_M)));
  if (e != cudaSuccess) return e;
  const long long grid = (a.npix + GRAD_THREADS - 1) / GRAD_THREADS;
  fn<<<(unsigned)grid, GRAD_THREADS, smem, s>>>(a, iters);
  return cudaGetLastError();
}

template <int K>
static cudaError_t launch_fit_m(const PixArgs& a, int iters, cudaStream_t s) {
  if (K <= 3) {
    switch (a.m) {
      case 4:
        return launch_fit_t<K, 4>(a, iters, s);
      case 5:
        return launch_fit_t<K, 5>(a, iters, s);
      case 10:
        return launch_fit_t<K, 10>(a, iters, s);
      case 20:
        return launch_fit_t<K, 20>(a, iters, s);
      case 32:
        return launch_fit_t<K, 32>(a, iters, s);
      default:
        break;
    }
  }
  return launch_fit_t<K, 0>(a, iters, s);
}

cudaError_t launch_fit(int K, const PixArgs& a, int iters, cudaStream_t s) {
  if (a.npix <= 0) return cudaSuccess;
  switch (K) {
    case 1:
      return launch_fit_m<1>(a, iters, s);
    case 2:
      return launch_fit_m<2>(a, iters, s);
    case 3:
      return launch_fit_m<3>(a, iters, s);
    case 4:
      return launch_fit_m<4>(a, iters, s);
    case 5:
      return launch_fit_m<5>(a, iters, s);
    case 6:
      return launch_fit_m<6>(a, iters, s);
    case 7:
      return launch_fit_m<7>(a, iters, s);
    case 8:
      return launch_fit_m<8>(a, iters, s);
    default:
      return cudaErrorInvalidValue;
  }
}

// K4: the harness update, elementwise over (pixel, k).
template <int K>
__global__ void __launch_bounds__(PX_THREADS) update_kernel(const PixArgs a) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npix) return;
#pragma unroll
  for (int k = 0; k < K; k++) {
    float tn, an;
    update_one(a, a.t_in[i * K + k], a.a_in[i * K + k], a.grad_t[i * K + k], a.grad_a[i * K + k], tn, an);
    a.t_out[i * K + k] = tn;
    a.a_out[i * K + k] = an;
  }
}

static int px_num_sms() { return num_sms_device(); }

template <int K, int M, int MODE>
static cudaError_t launch_px(const PixArgs& a, cudaStream_t s) {
  if (MODE == PX_UPDATE) {
    const long long grid = (a.npix + PX_THREADS - 1) / PX_THREADS;
    update_kernel<K><<<(unsigned)grid, PX_THREADS, 0, s>>>(a);
    return cudaGetLastError();
  }
  const int S = zstride(M ? M : (int)a.m);
  const int warps = PX_THREADS / 32;
  if (MODE == PX_EXPECTED) {
    const size_t smem = sizeof(float2) * warps * 32 * S;
    static SmemAttrOnce attr;
    cudaError_t e = smem_attr_once(attr, expected_kernel<K, M>, (int)(sizeof(float2) * warps * 32 * zstride(MAX_M)));
    if (e != cudaSuccess) return e;
    const long long grid = (a.npix + PX_THREADS - 1) / PX_THREADS;
    expected_kernel<K, M><<<(unsigned)grid, PX_THREADS, smem, s>>>(a);
    return cudaGetLastError();
  }
  const int gwarps = GRAD_THREADS / 32;
  const size_t smem = sizeof(float2) * gwarps * 32 * S;
  const int smem_max = (int)(sizeof(float2) * gwarps * 32 * zstride(MAX_M));
  if constexpr (M > 0 && M % 16 == 0) {
    if (((uintptr_t)a.z & 15u) == 0 && a.npix < (1ll << 31)) {
      PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
      if (enc) {
        CUtensorMap tm;
        const cuuint64_t gdim[2] = {(cuuint64_t)(2 * M), (cuuint64_t)a.npix};
        const cuuint64_t gstride[1] = {(cuuint64_t)(2 * M * sizeof(float))};
        const cuuint32_t box[2] = {32u, 32u}, estride[2] = {1u, 1u};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.z), gdim, gstride, box, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
          auto tfn = grad_kernel_tma<K, M, MODE>;
          const size_t tsmem = 1024 + (size_t)gwarps * (M / 16) * (4096 + 8);
          static SmemAttrOnce tattr;
          cudaError_t e = smem_attr_once(tattr, tfn, (int)tsmem);
          if (e != cudaSuccess) return e;
          long long grid = (a.npix + GRAD_THREADS - 1) / GRAD_THREADS;
          if (GRAD_PERSIST) {  // one wave
            static OccCache tocc;
            int per_sm = 0;
            e = occupancy_cached(tocc, tfn, GRAD_THREADS, tsmem, &per_sm);
            if (e != cudaSuccess) return e;
            const long long wave = (long long)per_sm * num_sms_device();
            if (wave > 0 && grid > wave) grid = wave;
          }
          // programmatic dependent launch: the CTAs of this step may be scheduled during the
          // previous kernel's tail (griddepcontrol.wait keeps every read behind its completion).
          // C5 L2-cold launch 18.1 -> 16.9 us, in the loop 13.57 -> 13.33 us.  SRT3D_PDL=0 disables.
          static const bool pdl = [] {
            const char* v = getenv("SRT3D_PDL");
            return !(v && v[0] == '0');
          }();
          if (pdl) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)grid);
            cfg.blockDim = dim3(GRAD_THREADS);
            cfg.dynamicSmemBytes = tsmem;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            e = cudaLaunchKernelEx(&cfg, tfn, a, tm);
            if (e != cudaSuccess) return e;
          } else {
            tfn<<<(unsigned)grid, GRAD_THREADS, tsmem, s>>>(a, tm);
          }
          return cudaGetLastError();
        }
      }
    }
  }
  auto fn = grad_kernel<K, M, MODE>;
  static SmemAttrOnce attr;
  cudaError_t e = smem_attr_once(attr, fn, smem_max);
  if (e != cudaSuccess) return e;
  const long long grid = (a.npix + GRAD_THREADS - 1) / GRAD_THREADS;
  fn<<<(unsigned)grid, GRAD_THREADS, smem, s>>>(a);
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
    case PX_GRAD:  // without a loss output the per-frequency |r|^2 accumulation is compiled out
      return a.loss ? launch_px_k<PX_GRAD>(K, a, s) : launch_px_k<PX_GRAD_NL>(K, a, s);
    case PX_GRAD_NL:
      return launch_px_k<PX_GRAD_NL>(K, a, s);
    case PX_GRAD_STEP:  // without a loss output the per-frequency |r|^2 accumulation is compiled out
      return a.loss ? launch_px_k<PX_GRAD_STEP>(K, a, s) : launch_px_k<PX_GRAD_STEP_NL>(K, a, s);
    case PX_GRAD_STEP_NL:
      return launch_px_k<PX_GRAD_STEP_NL>(K, a, s);
    case PX_UPDATE:
      return launch_px_k<PX_UPDATE>(K, a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace srt3d
