// K1 paired path (SRT3D_PATH_PAIRED) — photon -> sketch accumulator, Eq. (3)
// (PAPER.md:59-63), for pixels with hundreds of photons or more.
//
//   z[i][j-1] = (1/n_i) sum_p exp(i 2 pi j x_p / T),  j = j0+1 .. j0+M
//
// Why a second direct kernel: on sm_100a the direct sum is
// bound by register-file operand reads, not by FP32 lanes.  A packed FP32x2
// instruction costs max(2, #distinct even regs, #distinct odd regs) issue
// cycles, so the complex-power recurrence (FMUL2 + FFMA2 + FADD2) costs ~7
// cycles per (photon, j) per warp.  The rotated Chebyshev recurrence
// v_j = 2 cos(theta') v_{j-1} - v_{j-2} needs one FFMA2 + one FADD2 (~5
// cycles) — but only if the rotation class of every photon in an instruction
// is known at compile time: a photon with |sin theta| < |cos theta| runs its
// chain on theta' = theta + pi/2 (exact: i * w, keeps |sin theta'| >= 1/sqrt2,
// tools/sim_cheb_error.c) and its terms are rotated back by (-i)^j, which is a
// free operand swizzle (.LO_HI / negate) only when it is uniform.
//
// So each warp owns one pixel at a time and sorts the pixel's photons by
// class into two shared-memory queues (A: |sin| >= |cos|, no rotation;
// B: rotated).  Every step then processes one (A, B) pair per lane: slot x
// always class A, slot y always class B, an empty queue supplying the absent
// photon (zero table entry tab[T], zero seeds); two pairs per step (four
// independent chains per lane).  Photons are read with
// coalesced 16-byte loads (scalar head/tail peel to 16-byte alignment), the
// class of bin x is an integer test on u = 2x mod T (B iff 4u < T or 4u > 3T),
// and the warp-wide compaction is one packed shuffle scan per 256 photons.
// Per-lane fp32 sums are folded every <= 256 photons per lane with the fixed-order
// butterfly reduce-scatter (bitwise reproducible).
#include <cstdint>
#include <utility>

#include "sketch_impl.cuh"

namespace srt3d {

constexpr int PQ_CAP = 512;                  // photons per class queue per warp (power of two)
constexpr int PQ_SMEM_PER_WARP = 2 * (PQ_CAP + 8) * 2;  // + junk slots

template <int M>
struct PairAcc {
  u64 acc[M];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < M; j++) acc[j] = 0ull;
  }
  // Term J of the pass for two (A, B) pairs: advance the four chains (J > 0)
  // and accumulate xa0 + xa1 + (-i)^{1+J} (yb0 + yb1).
  template <int J>
  __device__ __forceinline__ void term(Chain& x0, Chain& y0, Chain& x1, Chain& y1) {
    if constexpr (J > 0) {
      x0.advance();
      y0.advance();
      x1.advance();
      y1.advance();
    }
    const u64 s0 = fadd2(x0.B, rot_back<J>(y0.B));
    const u64 s1 = fadd2(x1.B, rot_back<J>(y1.B));
    acc[J] = fadd2(acc[J], fadd2(s0, s1));
  }
  template <int... J>
  __device__ __forceinline__ void terms(std::integer_sequence<int, J...>, Chain& x0, Chain& y0, Chain& x1,
                                        Chain& y1) {
    (term<J>(x0, y0, x1, y1), ...);
  }
  // Chain seeds of photon x (T = absent) for the pass starting at j0 + 1;
  // rotated (class B) chains run on i * w.
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
  // Two (A, B) pairs: xa* class A (or T = absent), xb* class B (or T).
  __device__ __forceinline__ void pair2(const float2* tab, uint32_t xa0, uint32_t xb0, uint32_t xa1, uint32_t xb1,
                                        uint32_t T, uint32_t j0, float invT) {
    Chain x0 = seed<false>(tab, xa0, T, j0, invT), y0 = seed<true>(tab, xb0, T, j0, invT);
    Chain x1 = seed<false>(tab, xa1, T, j0, invT), y1 = seed<true>(tab, xb1, T, j0, invT);
    terms(std::make_integer_sequence<int, M>{}, x0, y0, x1, y1);
  }
};

// Warp-wide append of the 8 photons in v (valid iff `valid`) to the class
// queues; tA / tB are the warp-uniform tail counters.  Branch-free: invalid
// lanes write to the junk slot qA[PQ_CAP].
__device__ __forceinline__ void pq_append(uint16_t* qA, uint16_t* qB, const uint4 v, int nv, uint32_t T, int lane,
                                          uint32_t& tA, uint32_t& tB) {
  const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
  uint32_t isb = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const uint32_t x = (wv[i >> 1] >> (16 * (i & 1))) & 0xffffu;
    isb |= (class_b(x, T) ? 1u : 0u) << i;
  }
  const uint32_t vmask = nv >= 8 ? 0xffu : ((1u << nv) - 1u);
  isb &= vmask;
  const uint32_t nb = __popc(isb), na = (uint32_t)__popc(vmask) - nb;
  const uint32_t p = na | (nb << 16);
  uint32_t s = p;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, s, d);
    if (lane >= d) s += t;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, s, 31);
  const uint32_t ex = s - p;
  uint32_t oa = tA + (ex & 0xffffu), ob = tB + (ex >> 16);
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const uint16_t x = (uint16_t)((wv[i >> 1] >> (16 * (i & 1))) & 0xffffu);
    const bool b = (isb >> i) & 1u, ok = (vmask >> i) & 1u;
    uint16_t* dst = !ok ? qA + PQ_CAP : (b ? qB + (ob & (PQ_CAP - 1)) : qA + (oa & (PQ_CAP - 1)));
    *dst = x;
    oa += (ok && !b) ? 1u : 0u;
    ob += (ok && b) ? 1u : 0u;
  }
  tA += tot & 0xffffu;
  tB += tot >> 16;
}

template <int M>
__global__ void __launch_bounds__(SK_THREADS) sketch_pair_kernel(SketchArgs a) {
  extern __shared__ float2 tab[];
  build_phase_table(tab, a.T);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t* qA = reinterpret_cast<uint16_t*>(tab + ((a.T + 2) & ~1u)) + warp * 2 * (PQ_CAP + 8);
  uint16_t* qB = qA + PQ_CAP + 8;
  __syncthreads();

  constexpr int NV = 2 * M;
  constexpr int NVP = ((NV + 31) / 32) * 32;
  constexpr int VL = NVP / 32;
  constexpr int FLUSH_STEPS = 64;  // <= 256 photons per lane per fp32 partial
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const uint32_t off0 = (uint32_t)(((uintptr_t)a.bins >> 1) & 7u);
  const uint4* __restrict__ vb = reinterpret_cast<const uint4*>(a.bins - off0);
  const uint16_t* __restrict__ bins = a.bins;
  const uint32_t T = a.T, j0 = a.j0;
  const float invT = 1.0f / (float)a.T;

  for (long long pix = gw; pix < a.npix; pix += nw) {
    unsigned long long beg = a.offsets[pix], end = a.offsets[pix + 1];
    if (end < beg) end = beg;  // malformed CSR: empty
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
    uint32_t hA = 0, tA = 0, hB = 0, tB = 0;
    int since_flush = 0;
    PairAcc<M> pa;
    pa.zero();
    float res[VL];
#pragma unroll
    for (int i = 0; i < VL; i++) res[i] = 0.f;

    auto flush = [&]() {
      float f[NVP];
#pragma unroll
      for (int j = 0; j < M; j++) {
        f[2 * j] = lo_of(pa.acc[j]);
        f[2 * j + 1] = hi_of(pa.acc[j]);
      }
#pragma unroll
      for (int i = NV; i < NVP; i++) f[i] = 0.f;
      group_reduce_scatter<NVP, 32>(f, lane);
#pragma unroll
      for (int i = 0; i < VL; i++) res[i] += f[i];
      pa.zero();
      since_flush = 0;
    };
    // one step: lane takes entries (h + lane) and (h + 32 + lane) of each
    // queue if present (two (A, B) pairs, four chains)
    auto step = [&](bool useA, bool useB) {
      const uint32_t ia = hA + (uint32_t)lane, ib = hB + (uint32_t)lane;
      const uint32_t xa0 = (useA && ia < tA) ? (uint32_t)qA[ia & (PQ_CAP - 1)] : T;
      const uint32_t xb0 = (useB && ib < tB) ? (uint32_t)qB[ib & (PQ_CAP - 1)] : T;
      const uint32_t xa1 = (useA && ia + 32u < tA) ? (uint32_t)qA[(ia + 32u) & (PQ_CAP - 1)] : T;
      const uint32_t xb1 = (useB && ib + 32u < tB) ? (uint32_t)qB[(ib + 32u) & (PQ_CAP - 1)] : T;
      pa.pair2(tab, xa0, xb0, xa1, xb1, T, j0, invT);
      if (useA) hA = min(hA + 64u, tA);
      if (useB) hB = min(hB + 64u, tB);
      if (++since_flush >= FLUSH_STEPS) flush();
    };

    // scalar head + tail peel (< 8 photons each): one photon per lane
    {
      const int nh = (int)(hend - beg), nt = (int)(end - tbeg);
      const int nht = nh + nt;
      if (nht > 0) {
        uint4 v = make_uint4(0, 0, 0, 0);
        int nv = 0;
        if (lane < nht) {
          v.x = bins[lane < nh ? beg + lane : tbeg + (lane - nh)];
          nv = 1;
        }
        pq_append(qA, qB, v, nv, T, lane, tA, tB);
        __syncwarp();
      }
    }
    // Main loop with a single call site of the pair body (I-cache): pair
    // steps while both queues hold a full step, forced single-class steps when
    // a queue could overflow on the next round, else the next 16-byte round
    // (32 lanes x 8 photons), and at the end the remainder (absent partners).
    long long c = cb + lane;
    uint4 nxt = make_uint4(0, 0, 0, 0);
    if (c < ce) nxt = __ldcs(vb + c);
    for (;;) {
      const uint32_t na = tA - hA, nb = tB - hB;
      bool useA = true, useB = true;
      if (na >= 64u && nb >= 64u) {
      } else if (na > (uint32_t)(PQ_CAP - 256)) {
        useB = false;
      } else if (nb > (uint32_t)(PQ_CAP - 256)) {
        useA = false;
      } else if (c - lane < ce) {
        const uint4 v = nxt;
        const int nv = c < ce ? 8 : 0;
        if (c + 32 < ce) nxt = __ldcs(vb + c + 32);  // prefetch the lane's next chunk
        c += 32;
        __syncwarp();  // earlier steps are done reading the slots being overwritten
        pq_append(qA, qB, v, nv, T, lane, tA, tB);
        __syncwarp();
        continue;
      } else if (na == 0u && nb == 0u) {
        break;
      }
      step(useA, useB);
    }
    flush();
    const unsigned long long n = end - beg;
    const float inv = n ? 1.0f / (float)n : 0.0f;
    float* zrow = a.z + ((size_t)pix * a.mstride + j0) * 2;
#pragma unroll
    for (int i = 0; i < VL; i++) {
      const int idx = lane * VL + i;
      if (idx < NV) zrow[idx] = res[i] * inv;
    }
    __syncwarp();
  }
}

template <int M>
static cudaError_t launch_pair_t(const SketchArgs& a, cudaStream_t s, int num_sms) {
  auto fn = sketch_pair_kernel<M>;
  const size_t smem = sizeof(float2) * (((size_t)a.T + 2) & ~(size_t)1) + (size_t)(SK_THREADS / 32) * PQ_SMEM_PER_WARP;
  static bool attr_set = false;  // benign race: idempotent attribute set
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(SK_MAX_SMEM + 16 + (SK_THREADS / 32) * PQ_SMEM_PER_WARP));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static OccCache occ;
  int per_sm = 0;
  cudaError_t e = occupancy_cached(occ, fn, SK_THREADS, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long need = (a.npix + (SK_THREADS / 32) - 1) / (SK_THREADS / 32);
  long long grid = (long long)per_sm * num_sms;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  fn<<<(unsigned)grid, SK_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

size_t sketch_pair_smem(uint32_t T) {
  return sizeof(float2) * (((size_t)T + 2) & ~(size_t)1) + (size_t)(SK_THREADS / 32) * PQ_SMEM_PER_WARP;
}

cudaError_t launch_sketch_pair(int M, const SketchArgs& a, cudaStream_t s, int num_sms) {
  switch (M) {
#define SRT3D_CASE(MM) \
  case MM:             \
    return launch_pair_t<MM>(a, s, num_sms);
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
