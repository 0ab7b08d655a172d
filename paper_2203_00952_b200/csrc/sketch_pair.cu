// K1 class-sorted path (SRT3D_PATH_PAIRED) — photon -> sketch accumulator,
// Eq. (3), for pixels with hundreds of photons or more.
//
//   z[i][j-1] = (1/n_i) sum_p exp(i 2 pi j x_p / T),  j = j0+1 .. j0+M
//
// Why: on sm_100a the direct sum is bound by register-file
// operand reads, not by FP32 lanes.  A packed FP32x2 instruction costs
// max(2, #distinct even regs, #distinct odd regs) issue cycles, so the
// complex-power recurrence (FMUL2 + FFMA2 + FADD2) costs ~7 cycles per
// (photon, j) per warp.  The rotated Chebyshev recurrence
// v_j = 2 cos(theta') v_{j-1} - v_{j-2} needs one FFMA2 + one FADD2 (~5
// cycles) — if the rotation class of every photon in an instruction is known
// at compile time: a photon with |sin theta| < |cos theta| (class B) runs its
// chain on theta' = theta + pi/2 (exact: i * w, keeps |sin theta'| >= 1/sqrt2,
// tools/sim_cheb_error.c) and its terms must be rotated back by (-i)^j.
//
// The back-rotation is linear, so it need not be applied per photon: a lane
// that accumulates only class-B photons for a while can keep its accumulator
// in the "B frame" acc'_j = i^j acc_j, add the raw chain values, and rotate
// the whole accumulator back once (compile-time swizzles / negations per j).
// So each group of G = 4 lanes (one pixel, as the grouped kernel) stages a
// chunk of its pixel's photons (up to 256 + the head/tail peel) in shared
// memory partitioned by class — class A from the front, class B from the
// back, positions from a 4-lane shuffle scan of per-lane counts — then runs
// all class-A photons, switches the frame, runs all class-B photons, and
// switches back.  Both loops run the same class-uniform body (two photons
// per step, two FFMA2 + two FADD2 per term); the class of bin x is an
// integer test on u = 2x mod T (B iff 4u < T or 4u > 3T).  Per-lane fp32 sums
// are folded after every chunk (<= 68 photons per lane) with the fixed-order
// butterfly reduce-scatter (bitwise reproducible).
#include <cstdint>
#include <utility>

#include "sketch_impl.cuh"

namespace srt3d {

constexpr int SO_G = 4;                 // lanes per pixel
constexpr int SO_SLOTS = 32;            // 16-byte slots (8 photons) per chunk per group: 8 per lane
constexpr int SO_CAP = 328;             // staged photons per group: 256 + head/tail (< 16), padded so the
                                        // group buffers start 4 banks apart (164 words = 4 mod 32)
constexpr int SO_GROUPS = SK_THREADS / SO_G;
constexpr int SO_JUNK = SO_CAP - 1;     // store target of invalid photons (branch-free append)
constexpr int SO_BTOP = SO_CAP - 2;     // class B fills downwards from here

// class of bin x (x < T <= 65536): B iff 4u < T or 4u > 3T, u = 2x mod T
__device__ __forceinline__ uint32_t so_class_b(uint32_t x, uint32_t T) {
  const uint32_t u2 = 2u * x;
  const uint32_t u = min(u2, u2 - T);  // 2x mod T (the wrapped difference is larger when 2x < T)
  return (4u * u - T) > 2u * T ? 1u : 0u;
}

template <int M>
struct SortAcc {
  u64 acc[M];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < M; j++) acc[j] = 0ull;
  }
  template <int J>
  __device__ __forceinline__ void term(Chain& x, Chain& y) {
    if constexpr (J > 0) {
      x.advance();
      y.advance();
    }
    acc[J] = fadd2(acc[J], fadd2(x.B, y.B));
  }
  template <int... J>
  __device__ __forceinline__ void terms(std::integer_sequence<int, J...>, Chain& x, Chain& y) {
    (term<J>(x, y), ...);
  }
  // acc_J *= i^r with r = (1 + J) (to the B frame) or 3 (1 + J) (back), mod 4
  template <bool TO_B, int J>
  __device__ __forceinline__ void rot1() {
    constexpr int r = TO_B ? ((1 + J) & 3) : ((3 * (1 + J)) & 3);
    const u64 v = acc[J];
    if constexpr (r == 1) {
      acc[J] = pk(-hi_of(v), lo_of(v));
    } else if constexpr (r == 2) {
      acc[J] = neg2(v);
    } else if constexpr (r == 3) {
      acc[J] = pk(hi_of(v), -lo_of(v));
    }
  }
  template <bool TO_B, int... J>
  __device__ __forceinline__ void frame(std::integer_sequence<int, J...>) {
    (rot1<TO_B, J>(), ...);
  }
  // Chain seeds of photon x (T = absent: zero table entry, zero seeds) for the
  // pass starting at j0 + 1; class-B chains run on i * w.
  template <bool ROT>
  __device__ __forceinline__ static Chain seed(const float2* tab, uint32_t x, uint32_t T, uint32_t j0, float invT) {
    const float2 w = tab[x];
    Chain c;
    const float cc = ROT ? -2.f * w.y : 2.f * w.x;  // 2 cos(theta'), theta' = theta (+ pi/2)
    c.C2 = pk(cc, cc);
    if (j0 == 0) {
      c.A = pk(x < T ? 1.f : 0.f, 0.f);
      c.B = ROT ? pk(-w.y, w.x) : pk(w.x, w.y);
    } else {  // j0 = 32, 64, ...: i^{j0} = 1, i^{j0+1} = i
      const float2 a0 = tab[x < T ? phase_index(x, j0, T, invT) : T];
      const float2 a1 = tab[x < T ? phase_index(x, j0 + 1, T, invT) : T];
      c.A = pk(a0.x, a0.y);
      c.B = ROT ? pk(-a1.y, a1.x) : pk(a1.x, a1.y);
    }
    return c;
  }
  template <bool ROT>
  __device__ __forceinline__ void pair(const float2* tab, uint32_t x, uint32_t y, uint32_t T, uint32_t j0,
                                       float invT) {
    Chain cx = seed<ROT>(tab, x, T, j0, invT), cy = seed<ROT>(tab, y, T, j0, invT);
    terms(std::make_integer_sequence<int, M>{}, cx, cy);
  }
};

// Append the photons of v (bit i of vmask: photon i valid; valid photons
// first) to the group's class-partitioned buffer: class A at qb[fA ...),
// class B at qb[SO_BTOP-fB ...) downwards.  fA / fB are group-uniform fill
// counters.  Photon i goes to (B ? ob : oa + i) - (#B before i): no serial
// counter chain, one predicated store per photon.
__device__ __forceinline__ void so_append(uint16_t* qb, const uint4 v, uint32_t vmask, uint32_t T, int gl,
                                          uint32_t& fA, uint32_t& fB) {
  const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
  uint32_t isb = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) isb |= so_class_b(min((wv[i >> 1] >> (16 * (i & 1))) & 0xffffu, T), T) << i;
  isb &= vmask;
  const uint32_t nb = __popc(isb), na = (uint32_t)__popc(vmask) - nb;
  const uint32_t p = na | (nb << 16);
  uint32_t s = p;
  uint32_t t = __shfl_up_sync(0xffffffffu, s, 1, SO_G);
  if (gl >= 1) s += t;
  t = __shfl_up_sync(0xffffffffu, s, 2, SO_G);
  if (gl >= 2) s += t;
  const uint32_t tot = __shfl_sync(0xffffffffu, s, SO_G - 1, SO_G);
  const uint32_t ex = s - p;
  const uint32_t oa = fA + (ex & 0xffffu), ob = (uint32_t)SO_BTOP - fB - (ex >> 16);
#pragma unroll
  for (int i = 0; i < 8; i++) {  // unconditional store: invalid photons go to the junk slot
    const uint32_t nbefore = __popc(isb & ((1u << i) - 1u));
    const uint32_t dst = (((isb >> i) & 1u) ? ob : oa + (uint32_t)i) - nbefore;
    // bins >= T (precondition violation) become the absent photon T: zero table entry
    qb[((vmask >> i) & 1u) ? dst : (uint32_t)SO_JUNK] = (uint16_t)min((wv[i >> 1] >> (16 * (i & 1))) & 0xffffu, T);
  }
  fA += tot & 0xffffu;
  fB += tot >> 16;
}

template <int M>
__global__ void __launch_bounds__(SK_THREADS, 2) sketch_sorted_kernel(SketchArgs a) {
  extern __shared__ float2 tab[];
  build_phase_table(tab, a.T);
  const int lane = threadIdx.x & 31, gl = lane & (SO_G - 1), grp = lane / SO_G;
  uint16_t* qb = reinterpret_cast<uint16_t*>(tab + ((a.T + 2) & ~1u)) + (size_t)(threadIdx.x / SO_G) * SO_CAP;
  __syncthreads();

  constexpr int PPW = 32 / SO_G;
  constexpr int NV = 2 * M;
  constexpr int NVP = ((NV + SO_G - 1) / SO_G) * SO_G;
  constexpr int VL = NVP / SO_G;
  const long long warp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long ntiles = (a.npix + PPW - 1) / PPW;
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
    const int nh = (int)(hend - beg), nht = nh + (int)(end - tbeg);  // head/tail peel: < 16 photons
    // warp-uniform number of chunks
    int nck = (int)((ce - cb + SO_SLOTS - 1) / SO_SLOTS);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) nck = max(nck, __shfl_xor_sync(0xffffffffu, nck, d));
    if (nck == 0) nck = 1;

    float res[VL];
#pragma unroll
    for (int i = 0; i < VL; i++) res[i] = 0.f;
    SortAcc<M> sa;
    sa.zero();

    for (int k = 0; k < nck; k++) {
      // 1. stage the chunk, partitioned by class (two batches of four 16-byte
      // loads per lane in flight: register budget of 2 CTAs / SM)
      const long long s0 = cb + (long long)k * SO_SLOTS + gl;
      constexpr int QB = SO_SLOTS / SO_G / 2;
      uint4 v[QB];
#pragma unroll
      for (int q = 0; q < QB; q++) {
        const long long c = s0 + q * SO_G;
        v[q] = c < ce ? __ldcs(vb + c) : make_uint4(0, 0, 0, 0);
      }
      __syncwarp();  // the previous chunk's readers are done with qb
      uint32_t fA = 0, fB = 0;
      if (k == 0) {  // head/tail peel: up to 4 scalar photons per lane, one partial vector
        uint32_t hv[4] = {0, 0, 0, 0};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int idx = gl + q * SO_G;
          if (idx < nht) hv[q] = bins[idx < nh ? beg + idx : tbeg + (idx - nh)];
        }
        const int nq = min(4, max(0, (nht - gl + SO_G - 1) / SO_G));
        so_append(qb, make_uint4(hv[0] | (hv[1] << 16), hv[2] | (hv[3] << 16), 0, 0), (1u << nq) - 1u, T, gl, fA,
                  fB);
      }
#pragma unroll
      for (int h = 0; h < 2; h++) {
        uint4 w[QB];
#pragma unroll
        for (int q = 0; q < QB; q++) {
          w[q] = v[q];
          const long long c = s0 + (q + QB) * SO_G;
          if (h == 0) v[q] = c < ce ? __ldcs(vb + c) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < QB; q++) {
          const long long c = s0 + (q + h * QB) * SO_G;
          so_append(qb, w[q], c < ce ? 0xffu : 0u, T, gl, fA, fB);
        }
      }
      __syncwarp();
      // 2. class A (no rotation), two photons per step
#pragma unroll 1
      for (uint32_t i = gl; i < fA; i += 2 * SO_G) {
        const uint32_t x = qb[i];
        const uint32_t y = i + SO_G < fA ? (uint32_t)qb[i + SO_G] : T;
        sa.template pair<false>(tab, x, y, T, j0, invT);
      }
      // 3. class B in the rotated frame
      sa.template frame<true>(std::make_integer_sequence<int, M>{});
#pragma unroll 1
      for (uint32_t i = gl; i < fB; i += 2 * SO_G) {
        const uint32_t x = qb[SO_BTOP - i];
        const uint32_t y = i + SO_G < fB ? (uint32_t)qb[SO_BTOP - SO_G - i] : T;
        sa.template pair<true>(tab, x, y, T, j0, invT);
      }
      sa.template frame<false>(std::make_integer_sequence<int, M>{});
      // 4. fold every chunk (<= 68 photons per lane per fp32 partial; the
      // accumulators are dead while the next chunk is staged)
      {
        float f[NVP];
#pragma unroll
        for (int j = 0; j < M; j++) {
          f[2 * j] = lo_of(sa.acc[j]);
          f[2 * j + 1] = hi_of(sa.acc[j]);
        }
#pragma unroll
        for (int i = NV; i < NVP; i++) f[i] = 0.f;
        group_reduce_scatter<NVP, SO_G>(f, gl);
#pragma unroll
        for (int i = 0; i < VL; i++) res[i] += f[i];
        sa.zero();
      }
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

size_t sketch_pair_smem(uint32_t T) {
  return sizeof(float2) * (((size_t)T + 2) & ~(size_t)1) + (size_t)SO_GROUPS * SO_CAP * sizeof(uint16_t);
}

template <int M>
static cudaError_t launch_sorted_t(const SketchArgs& a, cudaStream_t s, int num_sms) {
  auto fn = sketch_sorted_kernel<M>;
  const size_t smem = sketch_pair_smem(a.T);
  static SmemAttrOnce attr;
  cudaError_t e = smem_attr_once(attr, fn, (int)sketch_pair_smem(SO_MAX_T));
  if (e != cudaSuccess) return e;
  static OccCache occ;
  int per_sm = 0;
  e = occupancy_cached(occ, fn, SK_THREADS, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  constexpr int PPW = 32 / SO_G;
  const long long tiles = (a.npix + PPW - 1) / PPW;
  const long long need = (tiles + (SK_THREADS / 32) - 1) / (SK_THREADS / 32);
  long long grid = (long long)per_sm * num_sms;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  fn<<<(unsigned)grid, SK_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sketch_pair(int M, const SketchArgs& a, cudaStream_t s, int num_sms) {
  switch (M) {
#define SRT3D_CASE(MM) \
  case MM:             \
    return launch_sorted_t<MM>(a, s, num_sms);
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
