#pragma once
// K1 — photon -> sketch accumulator, Eq. (3) on sm_100a.
//
//   z[i][j-1] = (1/n_i) sum_p exp(i 2 pi j x_p / T),  j = j0+1 .. j0+M
//
// Design:
//  * Each CTA first fills a shared-memory table tab[r] = exp(i 2 pi r / T),
//    r < T, rounded to fp32 from fp64 sincospi (exact-index phasors; the
//    index r = (j x) mod T is integer-exact).  The CTA is persistent and
//    reuses the table for every pixel it visits.
//  * A pixel is owned by a group of G lanes (G = 4, 8, 16 or 32; chosen from
//    the mean photons per pixel).  Photons are read as 16-byte vectors (8
//    uint16 bins per lane per load, coalesced across the group), after a
//    scalar head/tail peel that aligns the pixel's segment.
//  * Per photon x: w = tab[x], then the complex-power recurrence
//    p_j = p_{j-1} * w on the packed FP32x2 pipe (FMUL2 + FFMA2 per term) and
//    S_j += p_j (FADD2): 3 instructions / 6 FP32 lane-ops per (photon, j).
//    The worst-case fp32 drift over 32 steps from the exact w is 1.4e-6
//    (tools/sim_phasor_error.py), so no re-anchoring is needed for M <= 32;
//    m > 32 runs a second pass anchored at tab[(33 x) mod T].
//  * Accumulation is bounded: every super-chunk of <= 128 photons per lane is
//    folded across the group with a shuffle butterfly reduce-scatter (each
//    lane keeps 2M/G sums) into per-lane fp32 results.  The order is fixed,
//    so results are bitwise reproducible.
#include <cstdint>
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace srt3d {

// exp(i 2 pi r / T) for r < T into shared memory, fp64 sincospi on the
// centred index so the argument stays in (-1, 1]; tab[T] = 0 (absent photon).
__device__ __forceinline__ void build_phase_table(float2* tab, uint32_t T) {
  const double s = 2.0 / (double)T;
  for (uint32_t r = threadIdx.x; r <= T; r += blockDim.x) {
    if (r == T) {
      tab[r] = make_float2(0.f, 0.f);
      continue;
    }
    int rc = (2u * r > T) ? (int)r - (int)T : (int)r;
    double sn, cs;
    sincospi(s * (double)rc, &sn, &cs);
    tab[r] = make_float2((float)cs, (float)sn);
  }
}

// Exact phasor without a table (T too large for shared memory): fp64.
__device__ __forceinline__ float2 phasor_exact(uint32_t r, uint32_t T) {
  int rc = (2u * r > T) ? (int)r - (int)T : (int)r;
  double sn, cs;
  sincospi(2.0 * (double)rc / (double)T, &sn, &cs);
  return make_float2((float)cs, (float)sn);
}

// Multiply by i^n (n taken mod 4): exact (component swap / negation).
__device__ __forceinline__ float2 mul_ipow(float2 v, uint32_t n) {
  switch (n & 3u) {
    case 1: return make_float2(-v.y, v.x);
    case 2: return make_float2(-v.x, -v.y);
    case 3: return make_float2(v.y, -v.x);
    default: return v;
  }
}

// Per-lane accumulators of one pass (M frequencies) over a pixel's photons.
//
// SCH selects the phasor scheme for the terms j = j0+1 .. j0+M:
//  * SCH_CPOW: complex-power recurrence p_j = p_{j-1} * w (FMUL2 + FFMA2 per
//    term) + S_j += p_j (FADD2): 6 FP32 lane-ops per (photon, j).
//  * SCH_CHEB: rotated Chebyshev recurrence.  Both components of
//    v_j = e^{i j theta'} obey v_j = 2 cos(theta') v_{j-1} - v_{j-2}, one
//    FFMA2 per term (scalar broadcast coefficient, negated operand folded).
//    The recurrence is ill-conditioned where sin(theta') ~ 0 (the fp32
//    coefficient's rounding becomes an angle error delta / sin theta'), so a
//    photon whose base angle has |sin theta| < |cos theta| runs the chain on
//    theta' = theta + pi/2 (exact: i * w), |sin theta'| >= 1/sqrt 2, and its
//    terms are rotated back by (-i)^j — compile-time per j: nothing (j%4=0),
//    a sign (j%4=2, folded into an FFMA2 with a +-1 broadcast), or a
//    component swap with a sign (odd j: two selects on the ALU pipe).
//    4 FP32 lane-ops per (photon, j).  Worst-case phasor error 1.4e-6 for
//    j <= 32 and 2.8e-6 for j <= 64 at every T tested (tools/sim_cheb_error.c,
//    the same fp32 FMA sequence run for every x < T), equal to SCH_CPOW's.
// The table carries a zero entry at index T, used as the "absent photon"
// (keeps one copy of the unrolled body).
enum { SCH_CPOW = 0, SCH_CHEB = 1 };

template <int M, bool TAB, int SCH>
struct PhotonAcc {
  u64 acc[M];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < M; j++) acc[j] = 0ull;
  }
  // r >= T (a bin outside [0, T): precondition violation) reads the zero
  // entry tab[T] — unspecified but finite values, never an out-of-bounds read
  __device__ __forceinline__ static float2 base(const float2* tab, uint32_t r, uint32_t T) {
    if (TAB) return tab[min(r, T)];
    if (r >= T) return make_float2(0.f, 0.f);
    return phasor_exact(r, T);
  }

  // Two photons x, y as interleaved chains (ILP 2).  If !yvalid the second
  // chain contributes exactly 0 (zero base phasor / zero seeds).
  __device__ __forceinline__ void add2(const float2* tab, uint32_t x, uint32_t y, bool yvalid, uint32_t T,
                                       uint32_t j0, float invT) {
    const uint32_t yy = yvalid ? y : T;  // tab[T] = 0
    if (SCH != SCH_CPOW) {
      add2_cheb(tab, x, yy, yvalid, T, j0, invT);
      return;
    }
    const float2 w = base(tab, x, T), v = base(tab, yy, T);
    const u64 W = pk(w.x, w.y), Wn = pk(-w.y, w.x), V = pk(v.x, v.y), Vn = pk(-v.y, v.x);
    u64 P = W, Q = V;
    if (j0) {
      const float2 pa = base(tab, phase_index(x, j0 + 1, T, invT), T);
      const float2 qa = base(tab, yvalid ? phase_index(y, j0 + 1, T, invT) : T, T);
      P = pk(pa.x, pa.y);
      Q = pk(qa.x, qa.y);
    }
    acc[0] = fadd2(acc[0], fadd2(P, Q));
#pragma unroll
    for (int j = 1; j < M; j++) {
      P = cmul2(P, W, Wn);
      Q = cmul2(Q, V, Vn);
      acc[j] = fadd2(acc[j], fadd2(P, Q));
    }
  }

  // Per-photon constants of a rotated Chebyshev chain.
  struct ChebLane {
    u64 C2;  // (2 cos theta', 2 cos theta')
    u64 G2;  // (g, g), g = -1 if rotated else +1
    bool k;  // rotated by +pi/2
  };
  // Term J (0-based within the pass) of two chains: advance (J > 0) and
  // accumulate, rotated back by (-i)^{1+J} for a rotated chain.  A
  // compile-time index keeps the per-J code straight-line.
  template <int J>
  __device__ __forceinline__ void cheb_term(const ChebLane& X, const ChebLane& Y, u64& Ax, u64& Bx, u64& Ay,
                                            u64& By) {
    if constexpr (J > 0) {
      const u64 Nx = ffma2(Bx, X.C2, neg2(Ax));
      const u64 Ny = ffma2(By, Y.C2, neg2(Ay));
      Ax = Bx;
      Bx = Nx;
      Ay = By;
      By = Ny;
    }
    constexpr int rot = (1 + J) & 3;
    if constexpr (rot == 0) {
      acc[J] = fadd2(acc[J], fadd2(Bx, By));
    } else if constexpr (rot == 2) {
      acc[J] = ffma2(By, Y.G2, ffma2(Bx, X.G2, acc[J]));
    } else {  // rot 1: (-i) v = (s, -c); rot 3: (+i) v = (-s, c)
      constexpr float sg = rot == 1 ? 1.f : -1.f;
      const float bxr = lo_of(Bx), bxi = hi_of(Bx), byr = lo_of(By), byi = hi_of(By);
      const u64 Xr = pk(X.k ? sg * bxi : bxr, X.k ? -sg * bxr : bxi);
      const u64 Yr = pk(Y.k ? sg * byi : byr, Y.k ? -sg * byr : byi);
      acc[J] = fadd2(acc[J], fadd2(Xr, Yr));
    }
  }
  template <int... J>
  __device__ __forceinline__ void cheb_terms(std::integer_sequence<int, J...>, const ChebLane& X, const ChebLane& Y,
                                             u64& Ax, u64& Bx, u64& Ay, u64& By) {
    (cheb_term<J>(X, Y, Ax, Bx, Ay, By), ...);
  }

  // Rotated Chebyshev body (SCH_CHEB).  j0 must be a multiple of 4 (passes
  // are 32 wide), so the back-rotation (-i)^j depends on j - j0 only.
  __device__ __forceinline__ void add2_cheb(const float2* tab, uint32_t x, uint32_t yy, bool yvalid, uint32_t T,
                                            uint32_t j0, float invT) {
    const float2 w = base(tab, x, T), v = base(tab, yy, T);
    // SCH 2 (tools/sketch_tune.cu only): no rotation — wrong near sin = 0, used
    // to time the class-uniform body
    const bool kx = SCH == 2 ? false : fabsf(w.y) < fabsf(w.x), ky = SCH == 2 ? false : fabsf(v.y) < fabsf(v.x);
    // rotated bases e^{i theta'} = i^k w
    const float cx = kx ? -w.y : w.x, sx = kx ? w.x : w.y;
    const float cy = ky ? -v.y : v.x, sy = ky ? v.x : v.y;
    const float Cx = 2.f * cx, Cy = 2.f * cy;
    const float gx = kx ? -1.f : 1.f, gy = ky ? -1.f : 1.f;
    // seeds: (A, B) = (v_{j0}, v_{j0+1}) of each rotated chain
    u64 Ax, Bx, Ay, By;
    if (j0 == 0) {
      Ax = pk(1.f, 0.f);
      Bx = pk(cx, sx);
      Ay = pk(yvalid ? 1.f : 0.f, 0.f);
      By = pk(cy, sy);
    } else {
      const float2 a0 = mul_ipow(base(tab, phase_index(x, j0, T, invT), T), kx ? j0 : 0u);
      const float2 a1 = mul_ipow(base(tab, phase_index(x, j0 + 1, T, invT), T), kx ? j0 + 1 : 0u);
      const float2 b0 = mul_ipow(base(tab, yvalid ? phase_index(yy, j0, T, invT) : T, T), ky ? j0 : 0u);
      const float2 b1 = mul_ipow(base(tab, yvalid ? phase_index(yy, j0 + 1, T, invT) : T, T), ky ? j0 + 1 : 0u);
      Ax = pk(a0.x, a0.y);
      Bx = pk(a1.x, a1.y);
      Ay = pk(b0.x, b0.y);
      By = pk(b1.x, b1.y);
    }
    const ChebLane X{pk(Cx, Cx), pk(gx, gx), kx}, Y{pk(Cy, Cy), pk(gy, gy), ky};
    cheb_terms(std::make_integer_sequence<int, M>{}, X, Y, Ax, Bx, Ay, By);
  }
};

// ---- rotated Chebyshev helpers (paired path, bin-count DFT) ---------------
// Class of bin x: true = B (|sin theta| < |cos theta|, chain on theta + pi/2).
__device__ __forceinline__ bool class_b(uint32_t x, uint32_t T) {
  uint32_t u = 2u * x;
  u = u >= T ? u - T : u;  // 2x mod T (x < T)
  return 4u * u < T || 4u * u > 3u * T;
}

// Rotation of a class-B term back by (-i)^{1+J}: a compile-time operand
// swizzle / negation of the consuming FADD2.
template <int J>
__device__ __forceinline__ u64 rot_back(u64 y) {
  constexpr int rot = (1 + J) & 3;
  if constexpr (rot == 0) {
    return y;
  } else if constexpr (rot == 1) {  // (-i) v = (s, -c)
    return pk(hi_of(y), -lo_of(y));
  } else if constexpr (rot == 2) {
    return neg2(y);
  } else {  // (+i) v = (-s, c)
    return pk(-hi_of(y), lo_of(y));
  }
}

// One rotated Chebyshev chain: (A, B) = (v_{j-1}, v_j), C2 = (2 cos theta')^2.
struct Chain {
  u64 A, B, C2;
  __device__ __forceinline__ void advance() {
    const u64 N = ffma2(B, C2, neg2(A));
    A = B;
    B = N;
  }
};

// Butterfly reduce-scatter of NV floats over the G lanes of a group.  On
// return v[0 .. NV/G) of lane gl holds the group sums of the original
// entries [gl*NV/G, (gl+1)*NV/G).  Fixed order => deterministic.
template <int NV, int G>
__device__ __forceinline__ void group_reduce_scatter(float (&v)[NV], int gl) {
#pragma unroll
  for (int d = G / 2, n = NV; d >= 1; d >>= 1, n >>= 1) {
    const bool up = (gl & d) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; i++) {
      float send = up ? v[i] : v[i + n / 2];
      float keep = up ? v[i + n / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, d);
    }
  }
}

template <int M, int G, bool TAB, int SCH>
__global__ void __launch_bounds__(SK_THREADS) sketch_kernel(SketchArgs a) {
  extern __shared__ float2 tab[];
  if (sketch_regime_skip(a, M)) return;  // another candidate launch of this pass does the work
  if (TAB) {
    build_phase_table(tab, a.T);
    __syncthreads();
  }
  constexpr int PPW = 32 / G;                    // pixels per warp
  constexpr int NV = 2 * M;                      // floats per pixel
  constexpr int NVP = ((NV + G - 1) / G) * G;    // padded to a multiple of G
  constexpr int VL = NVP / G;                    // floats per lane after reduce-scatter
  constexpr int CPL = 16;                        // 16B chunks per lane per super-chunk (128 photons)
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const long long warp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long ntiles = (a.npix + PPW - 1) / PPW;
  // bins pointer is 2-byte aligned; slot s = p + off0 is 16-byte aligned when s % 8 == 0
  const uint32_t off0 = (uint32_t)(((uintptr_t)a.bins >> 1) & 7u);
  const uint4* __restrict__ vb = reinterpret_cast<const uint4*>(a.bins - off0);
  const uint16_t* __restrict__ bins = a.bins;
  const uint32_t T = a.T, j0 = a.j0;
  const float invT = 1.0f / (float)a.T;

  for (long long tile = warp0; tile < ntiles; tile += nwarps) {
    const long long pix = tile * PPW + grp;
    const bool valid = pix < a.npix;
    unsigned long long beg = 0, end = 0;
    if (valid) {
      beg = a.offsets[pix];
      end = a.offsets[pix + 1];
      if (end < beg) end = beg;  // malformed CSR: treat as empty (never read out of range)
    }
    // aligned body in slot space (slot = photon index + off0; 16B aligned when % 8 == 0)
    const unsigned long long asb = (beg + off0 + 7u) & ~7ull;
    const unsigned long long ase = (end + off0) & ~7ull;
    unsigned long long hend = end, tbeg = end;
    long long cb = 0, ce = 0;
    if (asb < ase) {
      hend = asb - off0;
      tbeg = ase - off0;
      cb = (long long)(asb >> 3);
      ce = (long long)(ase >> 3);
    }
    PhotonAcc<M, TAB, SCH> pa;
    pa.zero();
    // scalar head + tail peel (< 8 photons each), processed in pairs through
    // the same add2 body as the vector loop
    {
      const int nh = (int)(hend - beg), nt = (int)(end - tbeg), nht = nh + nt;
      for (int idx = gl; idx < nht; idx += 2 * G) {
        const int idy = idx + G;
        const unsigned long long px = idx < nh ? beg + idx : tbeg + (idx - nh);
        const bool yv = idy < nht;
        const unsigned long long py = yv ? (idy < nh ? beg + idy : tbeg + (idy - nh)) : px;
        pa.add2(tab, bins[px], bins[py], yv, T, j0, invT);
      }
    }

    // warp-uniform number of super-chunks
    const long long nchunks = ce - cb;
    int nsc = (int)((nchunks + (long long)G * CPL - 1) / ((long long)G * CPL));
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) nsc = max(nsc, __shfl_xor_sync(0xffffffffu, nsc, d));
    if (nsc == 0) nsc = 1;

    float res[VL];
#pragma unroll
    for (int i = 0; i < VL; i++) res[i] = 0.f;

    for (int sc = 0; sc < nsc; sc++) {
      const long long cend = min(ce, cb + (long long)(sc + 1) * G * CPL);
      long long c = cb + (long long)sc * G * CPL + gl;
      uint4 nxt = make_uint4(0, 0, 0, 0);
      if (c < cend) nxt = __ldg(vb + c);
#pragma unroll 1
      for (; c < cend; c += G) {
        const uint4 v = nxt;
        if (c + G < cend) nxt = __ldg(vb + c + G);  // prefetch the lane's next 16B chunk
#pragma unroll 1
        for (int h = 0; h < 4; h++) {
          const uint32_t wv = h == 0 ? v.x : (h == 1 ? v.y : (h == 2 ? v.z : v.w));
          pa.add2(tab, wv & 0xffffu, wv >> 16, true, T, j0, invT);
        }
      }
      float f[NVP];
#pragma unroll
      for (int j = 0; j < M; j++) {
        f[2 * j] = lo_of(pa.acc[j]);
        f[2 * j + 1] = hi_of(pa.acc[j]);
      }
#pragma unroll
      for (int i = NV; i < NVP; i++) f[i] = 0.f;
      group_reduce_scatter<NVP, G>(f, gl);
#pragma unroll
      for (int i = 0; i < VL; i++) res[i] += f[i];
      pa.zero();
    }
    if (valid) {
      const unsigned long long n = end - beg;
      const float inv = n ? 1.0f / (float)n : 0.0f;
      float* zrow = a.z + ((size_t)pix * a.mstride + j0) * 2;
#pragma unroll
      for (int i = 0; i < VL; i++) {
        const int idx = gl * VL + i;
        if (idx < NV) zrow[idx] = res[i] * inv;
      }
    }
  }
}

// ---- host-side dispatch ---------------------------------------------------
template <int M, int G, bool TAB, int SCH>
static cudaError_t launch_sketch_t(const SketchArgs& a, cudaStream_t s, int num_sms) {
  auto fn = sketch_kernel<M, G, TAB, SCH>;
  const size_t smem = TAB ? sizeof(float2) * (a.T + 1) : 0;
  static SmemAttrOnce attr;
  cudaError_t e = smem_attr_once(attr, fn, (int)SK_MAX_SMEM);
  if (e != cudaSuccess) return e;
  static OccCache occ;
  int per_sm = 0;
  e = occupancy_cached(occ, fn, SK_THREADS, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  constexpr int PPW = 32 / G;
  const long long tiles = (a.npix + PPW - 1) / PPW;
  const long long need = (tiles + (SK_THREADS / 32) - 1) / (SK_THREADS / 32);
  long long grid = (long long)per_sm * num_sms;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  fn<<<(unsigned)grid, SK_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

template <int G, bool TAB, int SCH>
static cudaError_t dispatch_m(int M, const SketchArgs& a, cudaStream_t s, int num_sms) {
  switch (M) {
#define SRT3D_CASE(MM) \
  case MM:             \
    return launch_sketch_t<MM, G, TAB, SCH>(a, s, num_sms);
    SRT3D_CASE(1) SRT3D_CASE(2) SRT3D_CASE(3) SRT3D_CASE(4) SRT3D_CASE(5) SRT3D_CASE(6) SRT3D_CASE(7) SRT3D_CASE(8)
    SRT3D_CASE(9) SRT3D_CASE(10) SRT3D_CASE(11) SRT3D_CASE(12) SRT3D_CASE(13) SRT3D_CASE(14) SRT3D_CASE(15)
    SRT3D_CASE(16) SRT3D_CASE(17) SRT3D_CASE(18) SRT3D_CASE(19) SRT3D_CASE(20) SRT3D_CASE(21) SRT3D_CASE(22)
    SRT3D_CASE(23) SRT3D_CASE(24) SRT3D_CASE(25) SRT3D_CASE(26) SRT3D_CASE(27) SRT3D_CASE(28) SRT3D_CASE(29)
    SRT3D_CASE(30) SRT3D_CASE(31) SRT3D_CASE(32)
#undef SRT3D_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace srt3d
