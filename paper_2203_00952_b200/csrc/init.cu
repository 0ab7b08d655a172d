// NEXT-3 — pixelwise initialisation of the sketched fit.
//
//   backprojection (matched filter), reading A18:
//     g_n = Re sum_{l=1..m} z_l hhat_l e^{-i omega_l t_n},  t_n = n T / N
//   greedy depths, reading A19: up to K local maxima of g
//     (g_n > 0, g_n > g_{n-1}, g_n >= g_{n+1}, circular), largest first (ties:
//     smallest n), each at circular grid distance d with d T >= min_sep N from
//     the earlier picks; sorted by depth; alpha = clamp(g / sum_l hhat_l^2, 0, 1);
//     unfilled slots t = (t_first + T/2) mod T, g = alpha = 0 (reading A14).
//
// One warp per pixel (persistent warps).  Each CTA first fills a shared table
// W[n] = exp(-i 2 pi n / N) (fp64 sincospi on the centred index, rounded once),
// so every grid phasor is exact to 1/2 ulp; the warp stages c_l = hhat_l z_l in
// shared memory and every lane evaluates 4 grid points at a time by Horner's
// rule in w = W[n] (two packed FFMA2 per (point, l), c_l broadcast from shared
// memory once per 4 points).  The greedy picking reads the warp's g row from
// shared memory; K rounds of a warp-wide argmax over the candidates.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace srt3d {

constexpr int BP_WARPS = 4;
constexpr int BP_PTS = 4;  // grid points per lane per Horner pass


__device__ __forceinline__ void fill_grid_table(float2* W, uint32_t N) {
  for (uint32_t n = threadIdx.x; n < N; n += blockDim.x) {
    const int nc = (2u * n > N) ? (int)n - (int)N : (int)n;
    double s, c;
    sincospi(-2.0 * (double)nc / (double)N, &s, &c);
    W[n] = make_float2((float)c, (float)s);
  }
}

// g at this lane's grid points of the pixel whose coefficients are in cs.
// PICK: into gbuf (shared), else to global g row.
template <bool PICK>
__device__ __forceinline__ void backproject_row(const float2* W, const float2* cs, uint32_t m, uint32_t N,
                                                float* grow, int lane) {
  for (uint32_t base = 0; base < N; base += 32 * BP_PTS) {
    u64 acc[BP_PTS], Wp[BP_PTS], Wn[BP_PTS];
#pragma unroll
    for (int q = 0; q < BP_PTS; q++) {
      uint32_t n = base + lane + 32 * q;
      n = n < N ? n : N - 1;
      const float2 w = W[n];
      Wp[q] = pk(w.x, w.y);
      Wn[q] = pk(-w.y, w.x);
      const float2 c = cs[m - 1];
      acc[q] = pk(c.x, c.y);
    }
    for (int l = (int)m - 2; l >= 0; l--) {
      const float2 c = cs[l];
      const u64 C = pk(c.x, c.y);
#pragma unroll
      for (int q = 0; q < BP_PTS; q++)  // acc = acc * w + c_l
        acc[q] = ffma2(pk(hi_of(acc[q]), hi_of(acc[q])), Wn[q], ffma2(pk(lo_of(acc[q]), lo_of(acc[q])), Wp[q], C));
    }
#pragma unroll
    for (int q = 0; q < BP_PTS; q++) {
      const uint32_t n = base + lane + 32 * q;
      const u64 S = cmul2(acc[q], Wp[q], Wn[q]);  // sum_l c_l w^l
      if (n < N) grow[n] = lo_of(S);
    }
  }
}

template <bool PICK>
__global__ void __launch_bounds__(BP_WARPS * 32) backproject_kernel(const BpArgs a) {
  extern __shared__ __align__(16) float2 bp_smem[];
  float2* W = bp_smem;                                    // [N]
  float2* cs_all = W + a.N;                               // [BP_WARPS][MAX_M]
  float* g_all = reinterpret_cast<float*>(cs_all + BP_WARPS * MAX_M);  // [BP_WARPS][N] (PICK)
  fill_grid_table(W, a.N);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2* cs = cs_all + warp * MAX_M;
  float* gbuf = g_all + (size_t)warp * a.N;
  const long long nw = (long long)gridDim.x * BP_WARPS;
  const uint32_t N = a.N, m = a.m;
  const float2* zg = reinterpret_cast<const float2*>(a.z);
  long long pix = (long long)blockIdx.x * BP_WARPS + warp;
  float2 zn0 = make_float2(0.f, 0.f), zn1 = zn0;  // the warp's next z row (m <= 64), prefetched
  if (pix < a.npix) {
    if ((uint32_t)lane < m) zn0 = zg[(size_t)pix * m + lane];
    if ((uint32_t)lane + 32 < m) zn1 = zg[(size_t)pix * m + lane + 32];
  }
  for (; pix < a.npix; pix += nw) {
    if ((uint32_t)lane < m) cs[lane] = make_float2(a.hh[lane] * zn0.x, a.hh[lane] * zn0.y);
    if ((uint32_t)lane + 32 < m) cs[lane + 32] = make_float2(a.hh[lane + 32] * zn1.x, a.hh[lane + 32] * zn1.y);
    if (pix + nw < a.npix) {
      if ((uint32_t)lane < m) zn0 = zg[(size_t)(pix + nw) * m + lane];
      if ((uint32_t)lane + 32 < m) zn1 = zg[(size_t)(pix + nw) * m + lane + 32];
    }
    __syncwarp();
    backproject_row<PICK>(W, cs, m, N, PICK ? gbuf : a.g + (size_t)pix * N, lane);
    __syncwarp();
    if (!PICK) continue;
    // greedy picks (identical rule and tie order to oracle/srt3d_ref.c).
    // Candidates (g_n > 0, g_n > g_{n-1}, g_n >= g_{n+1}) are found once and
    // kept as per-lane bit masks over the lane's points n = lane + 32 r
    // (r < N/32 <= 128); each round scans only the candidate bits.
    uint32_t cm[4];
#pragma unroll
    for (int w = 0; w < 4; w++) {
      cm[w] = 0u;
#pragma unroll 1
      for (uint32_t b = 0; b < 32; b++) {
        const uint32_t n = lane + 32u * (32u * w + b);
        if (n >= N) break;
        const float gv = gbuf[n];
        const float gp = gbuf[n == 0 ? N - 1 : n - 1], gn = gbuf[n + 1 == N ? 0 : n + 1];
        if (gv > 0.f && gv > gp && gv >= gn) cm[w] |= 1u << b;
      }
    }
    uint32_t pick[MAX_K];
    uint32_t c = 0;
    for (uint32_t k = 0; k < a.K; k++) {
      float best = 0.f;
      int bn = -1;
#pragma unroll
      for (int w = 0; w < 4; w++) {
        uint32_t bits = cm[w];
#pragma unroll 1
        while (bits) {
          const uint32_t b = __ffs(bits) - 1;
          bits &= bits - 1;
          const uint32_t n = lane + 32u * (32u * w + b);
          const float gv = gbuf[n];
          bool ok = true;
#pragma unroll 1
          for (uint32_t q = 0; q < c; q++) {
            uint32_t d = n > pick[q] ? n - pick[q] : pick[q] - n;
            d = min(d, N - d);
            if ((unsigned long long)d * a.T < (unsigned long long)a.min_sep * N) ok = false;
          }
          if (ok && (bn < 0 || gv > best)) {  // ascending n within the lane: ties keep the smaller n
            best = gv;
            bn = (int)n;
          }
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {  // warp argmax: larger g, then smaller n
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int on = __shfl_xor_sync(0xffffffffu, bn, o);
        if (on >= 0 && (bn < 0 || ob > best || (ob == best && on < bn))) {
          best = ob;
          bn = on;
        }
      }
      if (bn < 0) break;
      pick[c++] = (uint32_t)bn;
    }
    for (uint32_t x = 1; x < c; x++)  // sort by depth
      for (uint32_t y = x; y > 0 && pick[y - 1] > pick[y]; y--) {
        const uint32_t tmp = pick[y];
        pick[y] = pick[y - 1];
        pick[y - 1] = tmp;
      }
    const double tfirst = c ? (double)pick[0] * (double)a.T / (double)N : 0.0;
    for (uint32_t k = lane; k < a.K; k += 32) {
      const size_t o = (size_t)pix * a.K + k;
      const uint32_t pk_ = pick[k < c ? k : 0];
      if (k < c) {
        const float gv = gbuf[pk_];
        a.t_out[o] = (float)((double)pk_ * (double)a.T / (double)N);
        a.g_out[o] = gv;
        a.a_out[o] = fminf(fmaxf(gv * a.inv_sh2, 0.f), 1.f);
      } else {
        a.t_out[o] = (float)fmod(tfirst + 0.5 * (double)a.T, (double)a.T);
        a.g_out[o] = 0.f;
        a.a_out[o] = 0.f;
      }
    }
    if (lane == 0) a.count[pix] = (int32_t)c;
    __syncwarp();
  }
}

// K = 1 closed form (reading A20): t = (T / 2 pi) arg(z_1) in
// [0, T) (fp64 atan2 once per pixel), alpha = clamp(sum_j hhat_j Re(conj(p_j) z_j)
// / sum_j hhat_j^2, 0, 1) at that t with p_j = e^{i omega_j t} from the
// exact 32-bit fixed-point phase and the packed recurrence (as the gradient
// kernel).  A warp stages its 32 pixels' z rows (one contiguous slab) through
// shared memory with coalesced asynchronous copies (odd row stride:
// conflict-free per-thread row reads).
__global__ void __launch_bounds__(BP_WARPS * 32) init_k1_kernel(const BpArgs a) {
  extern __shared__ __align__(16) float2 k1_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t m = a.m, S = m | 1u;
  float2* tile = k1_smem + (size_t)warp * 32 * S;
  const long long row0 = ((long long)blockIdx.x * BP_WARPS + warp) * 32;
  if (row0 >= a.npix) return;
  const int nrows = (int)min(32ll, a.npix - row0);
  const float2* slab = reinterpret_cast<const float2*>(a.z) + (size_t)row0 * m;
  const uint32_t total = (uint32_t)nrows * m;
  uint32_t row = lane / m, col = lane - row * m;
  const uint32_t dq = 32 / m, dr = 32 - dq * m;
  for (uint32_t u = lane; u < total; u += 32) {  // all of the lane's copies in flight (LDGSTS)
    const unsigned d = (unsigned)__cvta_generic_to_shared(tile + row * S + col);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(slab + u) : "memory");
    col += dr;
    row += dq;
    if (col >= m) {
      col -= m;
      row++;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
  const long long pix = row0 + lane;
  if (lane >= nrows) return;
  const float2* zr = tile + lane * S;
  const float2 z1 = zr[0];
  float tf = 0.f, al = 0.f;
  if (hypot((double)z1.x, (double)z1.y) > 1e-12) {
    double t = (double)a.T * atan2((double)z1.y, (double)z1.x) / (2.0 * 3.14159265358979323846);
    if (t < 0.0) t += (double)a.T;
    tf = (float)t;
    if (tf >= (float)a.T) tf = 0.f;  // rounded up to T: the same point of the circle
    const uint32_t q = phase_q32(tf, 1.0 / (double)a.T);
    const float2 w = phasor_q32(q);
    const u64 W = pk(w.x, w.y), Wn = pk(-w.y, w.x);
    u64 P = W;
    float num = 0.f;
    for (uint32_t j = 0; j < m; j++) {
      if (j > 0) {
        if ((j & 31u) == 0) {
          const float2 p = phasor_q32(q * (j + 1));
          P = pk(p.x, p.y);
        } else {
          P = cmul2(P, W, Wn);
        }
      }
      const float2 zj = zr[j];
      num = fmaf(a.hh[j], fmaf(lo_of(P), zj.x, hi_of(P) * zj.y), num);  // hhat_j Re(conj(p_j) z_j)
    }
    al = fminf(fmaxf(num * a.inv_sh2, 0.f), 1.f);
  }
  a.t_out[pix] = tf;
  a.a_out[pix] = al;
}

// The same closed form with the warp's z slab staged by TMA (m % 16 == 0,
// m <= 64): one lane issues m/16 boxes of 32 rows x 32 floats (128-byte
// swizzle: 16-byte chunk c of row r at c ^ (r & 7), conflict-free per-thread
// row reads) on one mbarrier per box before anything else, so a warp's 8-16
// KB are in flight from its first instruction (the cp.async kernel above
// issues 32 8-byte copies per lane with their address arithmetic first);
// later boxes are awaited only when the frequency loop reaches them.  Rows
// past the frame end are zero-filled by the TMA unit.  Same arithmetic as
// init_k1_kernel, bit for bit.
constexpr int K1_WARPS = 4;
template <int NBOX>
__global__ void __launch_bounds__(K1_WARPS * 32) init_k1_tma_kernel(const BpArgs a,
                                                                    const __grid_constant__ CUtensorMap tm) {
  extern __shared__ unsigned char k1t_raw[];
  unsigned char* sm = k1t_raw + ((1024u - (smem_u32(k1t_raw) & 1023u)) & 1023u);  // 1 KB aligned (swizzle atoms)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* tile = sm + (size_t)warp * NBOX * 4096;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)K1_WARPS * NBOX * 4096) + warp * NBOX;
  const long long row0 = ((long long)blockIdx.x * K1_WARPS + warp) * 32;
  if (row0 >= a.npix) return;  // whole warp
  if (lane == 0) {
#pragma unroll
    for (int h = 0; h < NBOX; h++) mbar_init(bar + h, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int h = 0; h < NBOX; h++) {
      mbar_expect_tx(bar + h, 4096u);
      tma_load_2d(tile + h * 4096, &tm, h * 32, (int)row0, bar + h);
    }
  }
  __syncwarp();
  const int m = 16 * NBOX;
  const unsigned char* zr = tile + lane * 128;
  const int r7 = (lane & 7) << 4;
  auto zload = [&](int j) {  // z_j of this lane's row from box j / 16
    const float4 z2 = *reinterpret_cast<const float4*>(zr + (j / 16) * 4096 + ((((j % 16) / 2) << 4) ^ r7));
    return (j & 1) ? make_float2(z2.z, z2.w) : make_float2(z2.x, z2.y);
  };
  mbar_wait(bar, 0u);
  const float2 z1 = zload(0);
  float tf = 0.f, al = 0.f;
  const bool live = hypot((double)z1.x, (double)z1.y) > 1e-12;
  if (live) {
    double t = (double)a.T * atan2((double)z1.y, (double)z1.x) / (2.0 * 3.14159265358979323846);
    if (t < 0.0) t += (double)a.T;
    tf = (float)t;
    if (tf >= (float)a.T) tf = 0.f;  // rounded up to T: the same point of the circle
  }
  const uint32_t q = phase_q32(tf, 1.0 / (double)a.T);
  const float2 w = phasor_q32(q);
  const u64 W = pk(w.x, w.y), Wn = pk(-w.y, w.x);
  u64 P = W;
  float num = 0.f;
#pragma unroll
  for (int j = 0; j < m; j++) {
    if (j > 0 && j % 16 == 0) mbar_wait(bar + j / 16, 0u);  // every lane: the warp stays converged
    if (j > 0) {
      if ((j & 31) == 0) {
        const float2 p = phasor_q32(q * (uint32_t)(j + 1));
        P = pk(p.x, p.y);
      } else {
        P = cmul2(P, W, Wn);
      }
    }
    const float2 zj = zload(j);
    num = fmaf(a.hh[j], fmaf(lo_of(P), zj.x, hi_of(P) * zj.y), num);  // hhat_j Re(conj(p_j) z_j)
  }
  if (live) al = fminf(fmaxf(num * a.inv_sh2, 0.f), 1.f);
  const long long pix = row0 + lane;
  if (pix < a.npix) {
    a.t_out[pix] = tf;
    a.a_out[pix] = al;
  }
}

cudaError_t launch_init_k1(const BpArgs& a, cudaStream_t s) {
  if (a.npix <= 0) return cudaSuccess;
  // TMA staging where the shape allows it (SRT3D_INIT_K1_CPASYNC=1 forces the cp.async kernel: A/B and parity)
  const char* force = getenv("SRT3D_INIT_K1_CPASYNC");
  if (!(force && force[0] == '1') && a.m % 16 == 0 && a.m <= 64 && ((uintptr_t)a.z & 15u) == 0 &&
      a.npix < (1ll << 31)) {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    CUtensorMap tm;
    const cuuint64_t gdim[2] = {(cuuint64_t)(2 * a.m), (cuuint64_t)a.npix};
    const cuuint64_t gstride[1] = {(cuuint64_t)(2 * a.m * sizeof(float))};
    const cuuint32_t box[2] = {32u, 32u}, estride[2] = {1u, 1u};
    if (enc && enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.z), gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      const int nbox = (int)a.m / 16;
      void (*const fns[4])(const BpArgs, const CUtensorMap) = {init_k1_tma_kernel<1>, init_k1_tma_kernel<2>,
                                                                init_k1_tma_kernel<3>, init_k1_tma_kernel<4>};
      static SmemAttrOnce tattr[4];
      const size_t tsmem = 1024 + (size_t)K1_WARPS * nbox * (4096 + 8);
      cudaError_t e = smem_attr_once(tattr[nbox - 1], fns[nbox - 1], (int)tsmem);
      if (e != cudaSuccess) return e;
      const long long grid = (a.npix + 32 * K1_WARPS - 1) / (32 * K1_WARPS);
      fns[nbox - 1]<<<(unsigned)grid, K1_WARPS * 32, tsmem, s>>>(a, tm);
      return cudaGetLastError();
    }
  }
  const size_t smem = sizeof(float2) * BP_WARPS * 32 * (a.m | 1u);
  static SmemAttrOnce attr;
  cudaError_t e = smem_attr_once(attr, init_k1_kernel, (int)(sizeof(float2) * BP_WARPS * 32 * (MAX_M | 1)));
  if (e != cudaSuccess) return e;
  const long long grid = (a.npix + 32 * BP_WARPS - 1) / (32 * BP_WARPS);
  init_k1_kernel<<<(unsigned)grid, BP_WARPS * 32, smem, s>>>(a);
  return cudaGetLastError();
}

size_t backproject_smem(uint32_t N, bool pick) {
  return sizeof(float2) * ((size_t)N + BP_WARPS * MAX_M) + (pick ? sizeof(float) * BP_WARPS * (size_t)N : 0);
}

cudaError_t launch_backproject(const BpArgs& a, bool pick, cudaStream_t s, int num_sms) {
  if (a.npix <= 0) return cudaSuccess;
  // tensor-core path where the shape allows it (SRT3D_INIT_CUDA_CORES=1 forces
  // this kernel: A/B timing and parity of both paths)
  static const bool force_cores = [] {
    const char* e = getenv("SRT3D_INIT_CUDA_CORES");
    return e && e[0] == '1';
  }();
  if (!force_cores && backproject_tc_supported(a.N, a.m)) return launch_backproject_tc(a, pick, s, num_sms);
  const size_t smem = backproject_smem(a.N, pick);
  auto fn = pick ? backproject_kernel<true> : backproject_kernel<false>;
  static SmemAttrOnce attr[2];
  // the largest grid the entry points accept: N <= 8192 (backproject), N <= 4096 (picks)
  const size_t smem_cap = pick ? backproject_smem(4096, true) : backproject_smem(8192, false);
  cudaError_t e = smem_attr_once(attr[pick], fn, (int)smem_cap);
  if (e != cudaSuccess) return e;
  static OccCache occ[2];
  int per_sm = 0;
  e = occupancy_cached(occ[pick], fn, BP_WARPS * 32, smem, &per_sm);
  if (e != cudaSuccess) return e;
  long long grid = (a.npix + BP_WARPS - 1) / BP_WARPS;
  const long long cap = (long long)per_sm * num_sms;
  if (grid > cap) grid = cap;
  fn<<<(unsigned)grid, BP_WARPS * 32, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace srt3d
