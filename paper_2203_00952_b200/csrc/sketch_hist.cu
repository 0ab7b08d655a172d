// K5 — bin-count sketch path for pixels with many
// photons (n >~ T):  Eq. (3) regrouped by time bin,
//
//   z_j = (1/n) sum_{x=0}^{T-1} h[x] exp(i 2 pi j x / T),   h[x] = #{p : x_p = x}
//
// which is the same sum in a different order (counts are exact integers), so
// the result matches the direct path to rounding.  One
// persistent CTA per pixel at a time:
//   1. zero a shared uint32 histogram of T bins;
//   2. stream the pixel's photons with 16-byte vector loads (8 in flight per
//      thread) and count them with shared-memory atomics — 2 B of HBM per
//      photon, no FP32 work: this is the HBM-bound phase;
//   3. DFT of the histogram: thread t takes bins x = t, t+B, ..., weight h[x],
//      rotated Chebyshev recurrence over j with the bin's rotation class
//      known per branch (T*M terms per pixel instead of n*M; 1 FFMA2 + 1 FADD2
//      per term, DESIGN.md §5.0/§5.3);
//   4. fixed-order block reduction (warp reduce-scatter + smem), scale by 1/n.
#include <cstdint>
#include <utility>

#include "sketch_impl.cuh"

namespace srt3d {

#ifndef HS_DEFAULT_THREADS
#define HS_DEFAULT_THREADS 512  // CTA size (tools/hist_tune.cu)
#define HS_DEFAULT_UNROLL 8     // 16-byte loads in flight per thread
#endif

// acc[J] += h * e^{i 2 pi (j0 + 1 + J) x / T}, J < M, by the rotated
// Chebyshev chain of bin x (ROT: class B, chain on i*w, rotated back).
template <int M, bool ROT, int J>
__device__ __forceinline__ void dft_term(u64 (&acc)[M], Chain& c) {
  if constexpr (J > 0) c.advance();
  acc[J] = fadd2(acc[J], ROT ? rot_back<J>(c.B) : c.B);
}
template <int M, bool ROT, int... J>
__device__ __forceinline__ void dft_terms(u64 (&acc)[M], Chain& c, std::integer_sequence<int, J...>) {
  (dft_term<M, ROT, J>(acc, c), ...);
}
template <int M, bool ROT>
__device__ __forceinline__ void dft_bin(u64 (&acc)[M], const float2* tab, uint32_t x, float h, uint32_t T,
                                        uint32_t j0, float invT) {
  const float2 w = tab[x];
  Chain c;
  const float cc = ROT ? -2.f * w.y : 2.f * w.x;  // 2 cos(theta'), theta' = theta (+ pi/2)
  c.C2 = pk(cc, cc);
  if (j0 == 0) {
    c.A = pk(h, 0.f);
    c.B = ROT ? pk(-h * w.y, h * w.x) : pk(h * w.x, h * w.y);
  } else {  // j0 = 32, 64, ...: i^{j0} = 1, i^{j0+1} = i
    const float2 a0 = tab[phase_index(x, j0, T, invT)];
    const float2 a1 = tab[phase_index(x, j0 + 1, T, invT)];
    c.A = pk(h * a0.x, h * a0.y);
    c.B = ROT ? pk(-h * a1.y, h * a1.x) : pk(h * a1.x, h * a1.y);
  }
  dft_terms<M, ROT>(acc, c, std::make_integer_sequence<int, M>{});
}

template <int M, int HS_THREADS, int HS_UNROLL>
__global__ void __launch_bounds__(HS_THREADS) sketch_hist_kernel(SketchArgs a) {
  constexpr int NWARP = HS_THREADS / 32;
  constexpr int NV = 2 * M;
  constexpr int NVP = ((NV + 31) / 32) * 32;
  constexpr int VL = NVP / 32;
  extern __shared__ float2 tab[];
  const uint32_t T = a.T, j0 = a.j0;
  // hist[T] is a dump slot for out-of-range bins (precondition violations
  // count there and are never read back)
  uint32_t* hist = reinterpret_cast<uint32_t*>(tab + T + 1);
  float* red = reinterpret_cast<float*>(hist + ((T + 4) & ~3u));
  if (sketch_regime_skip(a, M)) return;  // another candidate launch of this pass does the work
  build_phase_table(tab, T);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float invT = 1.0f / (float)T;
  const uint32_t off0 = (uint32_t)(((uintptr_t)a.bins >> 1) & 7u);
  const uint4* __restrict__ vb = reinterpret_cast<const uint4*>(a.bins - off0);
  const uint16_t* __restrict__ bins = a.bins;

  for (uint32_t x = tid; x < T; x += HS_THREADS) hist[x] = 0u;  // later re-zeroed by the DFT pass
  for (long long pix = blockIdx.x; pix < a.npix; pix += gridDim.x) {
    __syncthreads();  // table build / previous pixel's DFT (which re-zeroes hist) done
    unsigned long long beg = a.offsets[pix], end = a.offsets[pix + 1];
    if (end < beg) end = beg;
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
    const int nh = (int)(hend - beg), nt = (int)(end - tbeg);
    if (tid < nh) atomicAdd(&hist[min((uint32_t)bins[beg + tid], T)], 1u);
    else if (tid < nh + nt) atomicAdd(&hist[min((uint32_t)bins[tbeg + (tid - nh)], T)], 1u);
    // 16-byte chunks, HS_UNROLL loads in flight per thread: full rounds, then
    // one predicated round (any photon count keeps its loads in flight)
    long long c = cb + tid;
    for (; c + (HS_UNROLL - 1) * HS_THREADS < ce; c += HS_UNROLL * HS_THREADS) {
      uint4 v[HS_UNROLL];
#pragma unroll
      for (int u = 0; u < HS_UNROLL; u++) v[u] = __ldcs(vb + c + u * HS_THREADS);  // streamed once: evict-first
#pragma unroll
      for (int u = 0; u < HS_UNROLL; u++) {
        const uint32_t w4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int h = 0; h < 4; h++) {
          atomicAdd(&hist[min(w4[h] & 0xffffu, T)], 1u);
          atomicAdd(&hist[min(w4[h] >> 16, T)], 1u);
        }
      }
    }
    if (c < ce) {
      uint4 v[HS_UNROLL];
#pragma unroll
      for (int u = 0; u < HS_UNROLL; u++)
        v[u] = c + u * HS_THREADS < ce ? __ldcs(vb + c + u * HS_THREADS) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < HS_UNROLL; u++) {
        if (c + u * HS_THREADS >= ce) break;
        const uint32_t w4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int h = 0; h < 4; h++) {
          atomicAdd(&hist[min(w4[h] & 0xffffu, T)], 1u);
          atomicAdd(&hist[min(w4[h] >> 16, T)], 1u);
        }
      }
    }
    __syncthreads();

    // DFT of the histogram over this thread's bins: the rotated Chebyshev
    // recurrence (one FFMA2 per term).  The rotation class of bin x is a
    // function of x, so each branch below is class-uniform and its
    // back-rotation is a compile-time operand swizzle; consecutive bins share
    // a class except at four boundaries, so warps almost never diverge.
    u64 acc[M];
#pragma unroll
    for (int j = 0; j < M; j++) acc[j] = 0ull;
    for (uint32_t x = tid; x < T; x += HS_THREADS) {
      const float h = (float)hist[x];
      hist[x] = 0u;  // ready for the next pixel
      if (class_b(x, T))
        dft_bin<M, true>(acc, tab, x, h, T, j0, invT);
      else
        dft_bin<M, false>(acc, tab, x, h, T, j0, invT);
    }
    float f[NVP];
#pragma unroll
    for (int j = 0; j < M; j++) {
      f[2 * j] = lo_of(acc[j]);
      f[2 * j + 1] = hi_of(acc[j]);
    }
#pragma unroll
    for (int i = NV; i < NVP; i++) f[i] = 0.f;
    group_reduce_scatter<NVP, 32>(f, lane);
#pragma unroll
    for (int i = 0; i < VL; i++) red[warp * NVP + lane * VL + i] = f[i];
    __syncthreads();
    if (tid < NV) {
      float sum = 0.f;
#pragma unroll 4
      for (int w = 0; w < NWARP; w++) sum += red[w * NVP + tid];
      const unsigned long long n = end - beg;
      const float inv = n ? 1.0f / (float)n : 0.0f;
      a.z[((size_t)pix * a.mstride + j0) * 2 + tid] = sum * inv;
    }
    __syncthreads();  // red / hist reuse
  }
}

inline size_t sketch_hist_smem_t(uint32_t T, int M, int nthreads) {
  const int NVP = ((2 * M + 31) / 32) * 32;
  return sizeof(float2) * (T + 1) + sizeof(uint32_t) * ((T + 4) & ~3u) + sizeof(float) * (nthreads / 32) * NVP;
}

template <int M, int HS_THREADS = HS_DEFAULT_THREADS, int HS_UNROLL = HS_DEFAULT_UNROLL>
static cudaError_t launch_hist_t(const SketchArgs& a, cudaStream_t s, int num_sms) {
  auto fn = sketch_hist_kernel<M, HS_THREADS, HS_UNROLL>;
  const size_t smem = sketch_hist_smem_t(a.T, M, HS_THREADS);
  static SmemAttrOnce attr;
  cudaError_t e = smem_attr_once(attr, fn, 227 * 1024);
  if (e != cudaSuccess) return e;
  static OccCache occ;
  int per_sm = 0;
  e = occupancy_cached(occ, fn, HS_THREADS, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  long long grid = (long long)per_sm * num_sms;
  if (grid > a.npix) grid = a.npix;
  if (grid < 1) grid = 1;
  fn<<<(unsigned)grid, HS_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

#ifndef HS_NO_DISPATCH
size_t sketch_hist_smem(uint32_t T, int M) { return sketch_hist_smem_t(T, M, 512); }  // largest CTA variant

// CTA size by the mean photons per pixel (tools/hist_tune.cu on B200; the
// thresholds live in sketch_regime): large CTAs stream heavy pixels (n ~
// 1e5-1e6) best; for n ~ 1e4 the per-pixel DFT, reduction and barriers
// dominate and more, smaller CTAs per SM win (C3-like frame: 512 threads
// 1.37 ms, 128 threads 0.86 ms).
template <int M>
static cudaError_t launch_hist_m(const SketchArgs& a, int threads, cudaStream_t s, int num_sms) {
  if (threads == 128) return launch_hist_t<M, 128, 4>(a, s, num_sms);
  if (threads == 256) return launch_hist_t<M, 256, 8>(a, s, num_sms);
  return launch_hist_t<M, 512, 8>(a, s, num_sms);
}

cudaError_t launch_sketch_hist(int M, const SketchArgs& a, int threads, cudaStream_t s, int num_sms) {
  switch (M) {
#define SRT3D_CASE(MM) \
  case MM:             \
    return launch_hist_m<MM>(a, threads, s, num_sms);
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
#endif

}  // namespace srt3d
