// EXPERIMENT (not built into libsrt3d.so; with tools/experiments/classed_streaming.patch —
// `git apply` it and copy this file to paper_2203_00952_b200/csrc/ to rebuild — measured
// and not shipped, DESIGN.md §5.1 / §5.6).
// K1 class-phased sketch (srt3d_sketch_classed) — photon -> sketch
// accumulator, Eq. (3), on a CSR frame whose pixels list
// their class-A photons first (n_A[i] of them), as srt3d_bucket_events_classed
// emits it.
//
//   z[i][j-1] = (1/n_i) sum_p exp(i 2 pi j x_p / T),  j = j0+1 .. j0+M
//
// Why: the rotated Chebyshev recurrence costs one FFMA2 +
// one FADD2 per (photon, j) only when every photon of an instruction has the
// same rotation class (class B: |sin theta| < |cos theta|, chain on
// theta + pi/2, terms rotated back by (-i)^j); with the class known per
// photon only at run time the back-rotation costs two selects per odd term and
// the body is no faster than the complex power, and sorting by class costs
// more than it saves unless the producer of the frame does it for free — the
// event bucketing keys its per-bucket sort by (pixel, class) at no extra pass.
// The grouped kernel (4 lanes per pixel, 16-byte vector loads, head/tail
// peel) runs the class-A range with unrotated chains and then the class-B
// range with rotated chains — the same class-uniform body, no selects; each
// fp32 partial is zeroed at a fold, so the B range's partials are rotated back
// (compile-time swizzles per j) just before their fold.  C5 frame: 1.49 vs
// 1.67 ms for srt3d_sketch.
#include <cstdint>
#include <type_traits>
#include <utility>

#include "sketch_impl.cuh"

namespace srt3d {

namespace {


// Class-uniform accumulator: two photons per step, rotated (ROT) or not.
template <int M>
struct ClsAcc {
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
  __device__ __forceinline__ void add2(const float2* tab, uint32_t x, uint32_t y, uint32_t T, uint32_t j0,
                                       float invT) {
    Chain cx = seed<ROT>(tab, x, T, j0, invT), cy = seed<ROT>(tab, y, T, j0, invT);
    terms(std::make_integer_sequence<int, M>{}, cx, cy);
  }
  template <int... J>
  __device__ __forceinline__ void rotate_back(std::integer_sequence<int, J...>) {
    ((acc[J] = rot_back<J>(acc[J])), ...);
  }
};

template <int M, int G>
__global__ void __launch_bounds__(SK_THREADS, 2) sketch_cls_kernel(SketchArgs a, const uint16_t* __restrict__ sbins,
                                                                  const uint32_t* __restrict__ nA) {
  extern __shared__ float2 tab[];
  build_phase_table(tab, a.T);
  __syncthreads();
  constexpr int PPW = 32 / G;
  constexpr int NV = 2 * M;
  constexpr int NVP = ((NV + G - 1) / G) * G;
  constexpr int VL = NVP / G;
  constexpr int CPL = 16;  // 16-byte chunks per lane per fold (128 photons)
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  const long long warp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long ntiles = (a.npix + PPW - 1) / PPW;
  const uint16_t* __restrict__ sb = sbins;  // the class-ordered CSR bins, indexed by the frame's offsets
  const uint32_t off0 = (uint32_t)(((uintptr_t)sb >> 1) & 7u);
  const uint4* __restrict__ vb = reinterpret_cast<const uint4*>(sb - off0);
  const uint32_t T = a.T, j0 = a.j0;
  const float invT = 1.0f / (float)a.T;

  for (long long tile = warp0; tile < ntiles; tile += nwarps) {
    const long long pix = tile * PPW + grp;
    const bool valid = pix < a.npix;
    unsigned long long beg = 0, end = 0, mid = 0;
    if (valid) {
      beg = a.offsets[pix];
      end = a.offsets[pix + 1];
      if (end < beg) end = beg;
      mid = beg + nA[pix];
      if (mid > end) mid = end;
    }
    float res[VL];
#pragma unroll
    for (int i = 0; i < VL; i++) res[i] = 0.f;
    ClsAcc<M> pa;
    pa.zero();
    auto fold = [&](bool rot) {
      if (rot) pa.rotate_back(std::make_integer_sequence<int, M>{});
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
    };
    // one class range [rb, re): head/tail peel in pairs, then 16-byte slots in
    // folds of CPL per lane; every fold count is warp-uniform
    auto range = [&](unsigned long long rb, unsigned long long re, auto rot_tag) {
      constexpr bool ROT = decltype(rot_tag)::value;
      const unsigned long long asb = (rb + off0 + 7u) & ~7ull, ase = (re + off0) & ~7ull;
      unsigned long long hend = re, tbeg = re;
      long long cb = 0, ce = 0;
      if (asb < ase) {
        hend = asb - off0;
        tbeg = ase - off0;
        cb = (long long)(asb >> 3);
        ce = (long long)(ase >> 3);
      }
      {
        const int nh = (int)(hend - rb), nht = nh + (int)(re - tbeg);
        for (int idx = gl; idx < nht; idx += 2 * G) {
          const int idy = idx + G;
          const uint32_t x = sb[idx < nh ? rb + idx : tbeg + (idx - nh)];
          const uint32_t y = idy < nht ? (uint32_t)sb[idy < nh ? rb + idy : tbeg + (idy - nh)] : T;
          pa.template add2<ROT>(tab, x, y, T, j0, invT);
        }
      }
      int nsc = (int)((ce - cb + (long long)G * CPL - 1) / ((long long)G * CPL));
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) nsc = max(nsc, __shfl_xor_sync(0xffffffffu, nsc, d));
      if (nsc == 0) nsc = 1;
      for (int sc = 0; sc < nsc; sc++) {
        const long long cend = min(ce, cb + (long long)(sc + 1) * G * CPL);
        long long c = cb + (long long)sc * G * CPL + gl;
        uint4 nxt = make_uint4(0, 0, 0, 0);
        if (c < cend) nxt = __ldcs(vb + c);
#pragma unroll 1
        for (; c < cend; c += G) {
          const uint4 v = nxt;
          if (c + G < cend) nxt = __ldcs(vb + c + G);
#pragma unroll 1
          for (int h = 0; h < 4; h++) {
            const uint32_t wv = h == 0 ? v.x : (h == 1 ? v.y : (h == 2 ? v.z : v.w));
            pa.template add2<ROT>(tab, wv & 0xffffu, wv >> 16, T, j0, invT);
          }
        }
        fold(ROT);
      }
    };
    range(beg, mid, std::false_type{});
    range(mid, end, std::true_type{});
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

template <int M>
cudaError_t launch_cls_t(const SketchArgs& a, const uint16_t* sbins, const uint32_t* nA, cudaStream_t s,
                         int num_sms) {
  constexpr int G = 4;
  auto fn = sketch_cls_kernel<M, G>;
  const size_t smem = sizeof(float2) * (a.T + 1);
  static bool attr_set = false;  // benign race: idempotent attribute set
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SK_MAX_SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static OccCache occ;
  int per_sm = 0;
  cudaError_t e = occupancy_cached(occ, fn, SK_THREADS, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  constexpr int PPW = 32 / G;
  const long long tiles = (a.npix + PPW - 1) / PPW;
  const long long need = (tiles + (SK_THREADS / 32) - 1) / (SK_THREADS / 32);
  long long grid = (long long)per_sm * num_sms;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  fn<<<(unsigned)grid, SK_THREADS, smem, s>>>(a, sbins, nA);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_sketch_cls(int M, const SketchArgs& a, const uint16_t* sbins, const uint32_t* nA, cudaStream_t s,
                              int num_sms) {
  switch (M) {
#define SRT3D_CASE(MM) \
  case MM:             \
    return launch_cls_t<MM>(a, sbins, nA, s, num_sms);
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
