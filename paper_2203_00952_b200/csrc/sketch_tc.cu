// K6 — tensor-core sketch, Eq. (3) regrouped
// by bin and factored once (a radix-Kb Cooley–Tukey step):
//
//   z_ij = (1/n_i) sum_p e^{i w_j x_p}                           (Eq. 3, w_j = 2 pi j / T)
//        = (1/n_i) sum_x h_i[x] e^{i w_j x}                        (h_i: photon counts per bin)
//   x = Kb a + b  (0 <= b < Kb, 0 <= a < R = ceil(T / Kb) <= 32):
//        = (1/n_i) sum_a e^{i w_j Kb a} [ sum_b h_i[a][b] e^{i w_j b} ]
//        = (1/n_i) sum_a W[a][j] P_i[a][j],   P_i = H_i V   (H_i: R x Kb, V: Kb x m)
//
// P = H V is a dense contraction over b with one V for every pixel and row:
// it runs on the 5th-generation tensor cores (tcgen05.mma kind::f16, M = 128
// rows = 4 pixels x 32 rows a, N = 4 MP columns, K = Kb), the twiddle by W and
// the sum over a on the CUDA cores in the epilogue (a warp per pixel: lane = a).
//
// Exactness of the operands:
//  * H: integer counts c < 2048 held as the raw bits of an fp16 number.  The
//    fp16 subnormal / first-normal binade is linear in its bit pattern:
//    bits c encode exactly c * 2^-24 for 0 <= c < 2048, so the shared-memory
//    histogram is built with plain integer atomics on packed u16 pairs.  Fed
//    to the MMA as is, a count below 1024 is a subnormal whose exponent field
//    overstates its magnitude by 2^(10 - log2 c), and the tensor core aligns
//    the products of a dot product by their exponent fields: the sum kept only
//    ~14-15 bits below its largest term (round 2, measured: a two-photon pixel
//    off by 1.3e-5, tools/tc_pair_probe.py).  So each unit's block is first
//    scaled in place by one exact HMUL2 by 2^10 per count pair (c 2^-14, a
//    normal fp16) and the epilogue multiplies by 2^14 (TC_NORMAL_COUNTS).
//    A pixel with more than CNT_MAX photons is split into rounds of at most
//    CNT_MAX photons whose MMAs accumulate into the same TMEM columns, so no
//    count ever reaches 2048.
//  * V = cos / sin (w_j b) from the exact phase index (j b) mod T in fp64,
//    split V = hi + 2^-12 lo with hi = fp16(V), lo = fp16(2^12 (V - hi)):
//    |V - hi - 2^-12 lo| <= 2^-24 (6e-8).  B = [cos hi | sin hi | cos lo |
//    sin lo] (N = 4 MP columns); products are exact in the fp32 accumulator.
//  * W[a][j] = e^{i w_j Kb a} from the exact phase index (j Kb a) mod T in
//    fp64, rounded to fp32.
//
// Roles (one persistent CTA per SM, 8 epilogue + 4 TC_BLD_PER_SLOT builder + 1 MMA warps):
//  * builders (warps 8.., TC_BLD_PER_SLOT per pixel slot; with TC_TMEM_A slot k is
//    warps 8 + k, 12 + k, ... so that warp % 4 is the slot's TMEM lane quarter):
//    per unit (a tile of 4 pixels, or one round of a heavy tile) scatter the
//    photons into the slot's shared-memory histogram with integer atomics
//    (16-byte vector loads of the tile's contiguous CSR range, issued after the
//    previous tile's scatter, two tiles ahead), then convert the counts to
//    normal fp16 (HMUL2 by 2^10) straight into TMEM A stage s with tcgen05.st,
//    zeroing the histogram as it is read, and arrive on full[s];
//  * the MMA warp, one thread: waits full[s] (and the TMEM accumulator's
//    accempty), issues Kb/16 tcgen05.mma with A from TMEM, commits to empty[s]
//    (A stage free) and, after a tile's last round, to accfull[tb];
//  * epilogue (warps 0..7: pixel slot w % 4, frequency half w / 4): reads its
//    accumulator columns, combines hi + lo, twiddles by W[lane],
//    reduce-scatters across the warp (lane l ends with frequency l), scales by
//    2^14 / n and stores z coalesced.
// Two TMEM A stages and two TMEM accumulators: the scatter of tile t + 1, the
// MMAs of tile t and the epilogue of tile t - 1 run concurrently.
// Supported: T <= TC_MAX_T (Kb <= 256, R <= 32), one pass of M <= 32
// frequencies (MP = 16 for M <= 16, else 32).
#include <cuda_fp16.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace srt3d {

namespace {

constexpr int TC_EPI_WARPS = 8;                 // two per pixel slot: warp w reads TMEM lanes 32 (w % 4), frequency half w / 4
#ifndef TC_BLD_PER_SLOT
#define TC_BLD_PER_SLOT 3  // builder warps per slot: 2 -> 4: C5 1.04 -> 0.94 ms (2: 96 regs; 5 spills, 1.26 ms);
                           // 4 -> 3 (80 regs, 672 threads): C5 0.883 -> 0.835-0.840 ms, C2 0.077 -> 0.078 ms
#endif
constexpr int TC_BLD_WARPS = 4 * TC_BLD_PER_SLOT;  // builder warps per pixel slot of a tile
constexpr int TC_SLOT_THREADS = 32 * TC_BLD_PER_SLOT;
constexpr int TC_MMA_WARP = TC_EPI_WARPS + TC_BLD_WARPS;
constexpr int TC_THREADS_ALL = (TC_MMA_WARP + 1) * 32;
constexpr uint32_t CNT_MAX = 2040;      // photons of one pixel per round: every count < 2048, <= 256 groups
// 16-byte photon groups per builder thread: a round's <= CNT_MAX photons span <= 256 groups
constexpr int PF = (256 + TC_SLOT_THREADS - 1) / TC_SLOT_THREADS;
// per-unit flags (builders -> MMA issuer, through shared memory under the full barrier)
constexpr uint32_t TC_TPC_MAX = 768;  // tiles per CTA per launch (offsets staged in shared memory)
constexpr uint32_t UF_FIRST = 1, UF_LAST = 2, UF_END = 4, UF_TB = 8;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major SWIZZLE_NONE operand: 8 x 16-byte core matrices (128 B each),
// LBO = 128 B between K-adjacent core matrices, SBO between 8-row groups
__device__ __forceinline__ uint64_t ns_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100); layout type 0 = SWIZZLE_NONE
  return d;
}

#ifndef TC_NORMAL_COUNTS
// 1: before its MMAs, each unit's histogram is converted in place from u16 counts (read by the
// MMA as fp16 subnormal bit patterns c 2^-24) to the normal fp16 values c 2^-14.  With subnormal counts the
// tensor core's accumulation keeps only ~13-14 bits below the largest product of a dot product
// (measured: photons sharing a row lose up to ~3e-5 per pair, tools/tc_pair_probe.py).
#define TC_NORMAL_COUNTS 1
#endif
#ifndef TC_LATE_PREFETCH
#define TC_LATE_PREFETCH 1
#endif
#ifndef TC_TMEM_A
// 1: the builders convert each unit's counts straight into a TMEM A stage (tcgen05.st) and zero the
// shared-memory histogram in the same pass; the MMAs read A from TMEM (the histogram is never an
// MMA operand, so one shared-memory stage suffices and the separate zeroing pass disappears)
#define TC_TMEM_A 1  // C5 0.936 -> 0.929 ms, C2 0.077 -> 0.066 ms (measured round 2)
#endif
#if defined(TC_CP) && TC_CP && TC_TMEM_A
#error "TC_CP (tcgen05.cp of shared-memory stages) and TC_TMEM_A (tcgen05.st of converted counts) exclude each other"
#endif
#ifndef TC_CP
// 1: each histogram stage copied into TMEM (tcgen05.cp 128x256b) and multiplied from there (A in
// TMEM: 98 instead of 127 cycles per MMA in isolation, microbench/umma_rate.cu).  Measured slower in
// the kernel: C5 0.91 vs 0.68 ms (the TMEM writes contend with the epilogue's TMEM reads); off.
#define TC_CP 0
#endif
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bd, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TCS_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra TCS_WAIT_%=;\n\t}" ::"r"(su32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; i++) v[i] = __uint_as_float(r[i]);
}

// Kb = K columns per row (power of two, 16..256) and its log2: 32 rows x Kb >= T
__host__ __device__ inline uint32_t tc_log2_kb(uint32_t T) {
  uint32_t q = 4;
  while ((32u << q) < T) q++;
  return q;
}

// The bin x of a photon IS its element index in its pixel's 32 x Kb block:
// with x's bits read as [a_hi (2) | k_hi (q - 3) | a_lo (3) | k_lo (3)] the
// block's K-major SWIZZLE_NONE layout [a_hi][k_hi][a_lo][k_lo] (row a = 8 a_hi
// + a_lo, column k = 8 k_hi + k_lo) puts bin x at fp16 element x, and
//   x = X_row(a) + X_col(k),  X_row(a) = 8 Kb a_hi + 8 a_lo,  X_col(k) = 64 k_hi + k_lo,
// so e^{i w x} = W[a] V[k] with W[a] = e^{i w X_row(a)}, V[k] = e^{i w X_col(k)}.
__host__ __device__ inline uint32_t tc_xrow(uint32_t a, uint32_t q) { return ((a >> 3) << (q + 3)) + ((a & 7u) << 3); }
__host__ __device__ inline uint32_t tc_xcol(uint32_t k) { return ((k >> 3) << 6) + (k & 7u); }

// a 16-byte photon group at aligned element index e0, only its elements inside [flo, fhi)
__device__ __noinline__ uint4 load_group_checked(const uint4* gp, uint32_t e0, uint32_t flo, uint32_t fhi) {
  if (e0 >= flo && e0 + 8u <= fhi) return __ldg(gp);
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  const uint16_t* e16 = reinterpret_cast<const uint16_t*>(gp);
#pragma unroll
  for (uint32_t e = 0; e < 8; e++)
    if (e0 + e >= flo && e0 + e < fhi) w[e >> 1] |= (uint32_t)__ldg(e16 + e) << ((e & 1u) * 16);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

#ifdef TC_PROF
// tools-only timing build (SRT3D_EXTRA=-DTC_PROF): per-role cycle counters summed over CTAs
__device__ unsigned long long tc_prof[16];
#define TCP_T0 const long long _tcp0 = clock64();
#define TCP_ADD(i, t0) atomicAdd(&tc_prof[i], (unsigned long long)(clock64() - (t0)))
#else
#define TCP_T0
#define TCP_ADD(i, t0)
#endif

template <int MP>
__global__ void __launch_bounds__(TC_THREADS_ALL, 1)
    sketch_tc_kernel(SketchArgs a, uint32_t M, long long pbase, long long pcount, uint32_t tpc) {
  extern __shared__ unsigned char tcs_raw[];
  if (sketch_regime_skip(a, (int)M)) return;  // another candidate launch of this pass does the work
  constexpr int N = 4 * MP;
  unsigned char* sm = tcs_raw + ((128u - (su32(tcs_raw) & 127u)) & 127u);
  const uint32_t T = a.T;
  const uint32_t q = tc_log2_kb(T), Kb = 1u << q;
  const uint32_t SLOT_B = 64u * Kb;          // bytes of one pixel's 32 x Kb fp16 block
  const uint32_t ASZ = 4u * SLOT_B;          // one A stage: 128 rows
  const uint32_t SBO = 16u * Kb;             // bytes between 8-row groups (A and B)
  unsigned char* A0 = sm;
  unsigned char* Bs = sm + 2 * ASZ;
  float2* Ws = reinterpret_cast<float2*>(Bs + (size_t)N * Kb * 2u);  // [MP][32] (frequency-major)
  uint32_t* so = reinterpret_cast<uint32_t*>(Ws + MP * 32);            // this CTA's offsets [4 ntl + 1]
  uint32_t* rounds_s = so + 4 * TC_TPC_MAX + 1;                         // rounds per local tile [ntl]
  __shared__ __align__(8) uint64_t full_bar[2], empty_bar[2], accfull_bar[2], accempty_bar[2], afree_bar[2];
  __shared__ uint32_t tmem_slot, uflags[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- one-time setup: B (hi | lo split), W, zeroed A stages, barriers, TMEM ----
  // V[k][j] = e^{i w_j X_col(k)}, X_col(k) = 64 k_hi + k_lo, as the fp64 product of
  // e^{i w_j 64 k_hi} and e^{i w_j k_lo} (40 sincospi per frequency instead of Kb; the
  // product's rounding, ~1e-16, is far below the fp16 hi/lo split's 2^-24), the factors staged
  // in the (not yet used) histogram region
  // (Kb >= 64: the region holds the 40 MP factors; smaller blocks take sincospi per entry)
  double2* vf = reinterpret_cast<double2*>(A0);  // [MP][40]: k_hi = 0..31, then k_lo = 0..7
  const bool vfact = 2u * ASZ >= (uint32_t)MP * 40u * (uint32_t)sizeof(double2);
  for (uint32_t e = tid; vfact && e < (uint32_t)MP * 40u; e += TC_THREADS_ALL) {
    const uint32_t jj = e / 40u, i = e % 40u;
    double2 v = make_double2(0.0, 0.0);
    if (jj < M && (i >= 32u || i < (Kb >> 3))) {
      const uint32_t j = a.j0 + 1u + jj;
      const uint32_t xc = i < 32u ? 64u * i : i - 32u;
      const uint32_t r = (uint32_t)(((unsigned long long)j * xc) % T);
      sincospi(2.0 * (double)r / (double)T, &v.y, &v.x);
    }
    vf[e] = v;
  }
  __syncthreads();
  for (uint32_t e = tid; e < (uint32_t)MP * Kb; e += TC_THREADS_ALL) {
    const uint32_t jj = e >> q, k = e & (Kb - 1u);
    __half h[4] = {__float2half(0.f), __float2half(0.f), __float2half(0.f), __float2half(0.f)};
    if (jj < M) {
      double c, sn;
      if (vfact) {
        const double2 ph = vf[jj * 40u + (k >> 3)], pl = vf[jj * 40u + 32u + (k & 7u)];
        c = ph.x * pl.x - ph.y * pl.y;
        sn = ph.x * pl.y + ph.y * pl.x;
      } else {
        const uint32_t r = (uint32_t)(((unsigned long long)(a.j0 + 1u + jj) * tc_xcol(k)) % T);
        sincospi(2.0 * (double)r / (double)T, &sn, &c);
      }
      const __half ch = __double2half(c), sh = __double2half(sn);
      h[0] = ch;
      h[1] = sh;
      h[2] = __double2half((c - (double)__half2float(ch)) * 4096.0);
      h[3] = __double2half((sn - (double)__half2float(sh)) * 4096.0);
    }
#pragma unroll
    for (int g = 0; g < 4; g++) {
      const uint32_t n = (uint32_t)g * MP + jj;
      *reinterpret_cast<__half*>(Bs + (n >> 3) * SBO + (k >> 3) * 128u + (n & 7u) * 16u + (k & 7u) * 2u) = h[g];
    }
  }
  for (uint32_t e = tid; e < (uint32_t)MP * 32u; e += TC_THREADS_ALL) {
    const uint32_t jj = e >> 5, ar = e & 31u, xr = tc_xrow(ar, q);
    float2 w = make_float2(0.f, 0.f);
    if (jj < M && xr < T) {
      const uint32_t j = a.j0 + 1u + jj;
      const uint32_t r = (uint32_t)(((unsigned long long)j * xr) % T);
      double sn, c;
      sincospi(2.0 * (double)r / (double)T, &sn, &c);
      w = make_float2((float)c, (float)sn);
    }
    Ws[e] = w;
  }
  __syncthreads();  // every V product read its factors before the histogram region is zeroed
  for (uint32_t e = tid; e < 2 * ASZ / 16; e += TC_THREADS_ALL)
    reinterpret_cast<uint4*>(A0)[e] = make_uint4(0u, 0u, 0u, 0u);
  // this CTA's tiles: [t0, t0 + ntl) of the launch's ceil(pcount / 4); its pixels' offsets staged
  // in shared memory (pixels past the launch's range repeat the last offset: empty)
  const long long ntiles = (pcount + 3) / 4;
  const long long t0 = (long long)blockIdx.x * tpc;
  const uint32_t ntl = (uint32_t)max(0ll, min((long long)tpc, ntiles - t0));
  const long long p0 = pbase + 4 * t0, pend = pbase + pcount;
  for (uint32_t i = tid; i <= 4 * ntl; i += TC_THREADS_ALL) so[i] = a.offsets[min(p0 + (long long)i, pend)];
  __syncthreads();
  for (uint32_t i = tid; i < ntl; i += TC_THREADS_ALL) {
    uint32_t mx = 0;
    for (int k = 0; k < 4; k++) mx = max(mx, so[4 * i + k + 1] - so[4 * i + k]);
    rounds_s[i] = mx == 0 ? 1u : (mx + CNT_MAX - 1) / CNT_MAX;
  }
  if (tid == 0) {
    for (int s = 0; s < 2; s++) {
      mbar_init(&full_bar[s], TC_BLD_WARPS);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&accfull_bar[s], 1);
      mbar_init(&accempty_bar[s], TC_EPI_WARPS);
      mbar_init(&afree_bar[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"((TC_CP || TC_TMEM_A) ? 512u : 2u * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp >= TC_EPI_WARPS && warp < TC_MMA_WARP) {
    // ======================= builders: warps 8 + B k .. 8 + B k + B - 1 own pixel slot k (B = TC_BLD_PER_SLOT) ====
#if TC_TMEM_A
    // slot k = builder warps 8 + k, 12 + k, ...: warp % 4 == k, the TMEM lane quarter of the slot's rows
    const uint32_t slot = (uint32_t)(warp - TC_EPI_WARPS) & 3u;
    const uint32_t wi = (uint32_t)(warp - TC_EPI_WARPS) >> 2;  // warp within the slot
    const uint32_t pt = wi * 32u + (uint32_t)lane;
#else
    const uint32_t slot = (uint32_t)(warp - TC_EPI_WARPS) / TC_BLD_PER_SLOT;
    const uint32_t pt = (uint32_t)(tid - TC_EPI_WARPS * 32) - slot * TC_SLOT_THREADS;
#endif
    const uint32_t esh = (uint32_t)(reinterpret_cast<uintptr_t>(a.bins) >> 1) & 7u;  // elements before 16 B alignment
    const uint4* gb = reinterpret_cast<const uint4*>(a.bins - esh);
    // the photon range [b0, b1) of this slot's pixel of local tile lt, round r
    auto range = [&](uint32_t lt, uint32_t r, uint32_t& b0, uint32_t& b1) {
      const uint32_t o0 = so[4 * lt + slot], o1 = so[4 * lt + slot + 1];
      b0 = min(o0 + r * CNT_MAX, o1);
      b1 = min(o1, b0 + CNT_MAX);
    };
    // the frame's photon range [offsets[0], offsets[npix]) in aligned element coordinates: a 16-byte
    // group straddling either end is read element by element (the header's promise: no read outside
    // it); only a pixel range starting in the frame's first or ending in its last group meets one
    const uint32_t flo = a.offsets[0] + esh, fhi = a.offsets[a.npix] + esh;
    auto load_groups = [&](uint32_t lt, uint32_t r, uint4 (&v)[PF]) {
      uint32_t b0, b1;
      range(lt, r, b0, b1);
      const uint32_t G0 = (b0 + esh) >> 3, G1 = (b1 + esh + 7u) >> 3;
      if (8u * G0 >= flo && 8u * G1 <= fhi) {
#pragma unroll
        for (int g = 0; g < PF; g++) {
          const uint32_t G = G0 + pt + (uint32_t)g * TC_SLOT_THREADS;
          v[g] = (b0 < b1 && G < G1) ? __ldg(gb + G) : make_uint4(0u, 0u, 0u, 0u);
        }
      } else {
        for (int g = 0; g < PF; g++) {
          const uint32_t G = G0 + pt + (uint32_t)g * TC_SLOT_THREADS;
          v[g] = (b0 < b1 && G < G1) ? load_group_checked(gb + G, 8u * G, flo, fhi) : make_uint4(0u, 0u, 0u, 0u);
        }
      }
    };
    uint32_t unit = 0;
    // one local tile: its rounds from `cur` (round 0 loaded two tiles earlier), tile lt + 2's
    // first round issued into `dst` (the buffer of tile lt - 1, consumed)
    auto body = [&](uint32_t lt, uint4 (&cur)[PF], uint4 (&dst)[PF]) {
      const uint32_t rounds = rounds_s[lt];
      for (uint32_t r = 0; r < rounds; r++, unit++) {
        const uint32_t s = unit & 1u;
        unsigned char* Ab = A0 + (TC_TMEM_A ? 0u : s * ASZ) + slot * SLOT_B;  // TMEM A: one histogram stage
        if (r > 0) load_groups(lt, r, cur);  // heavy pixel rounds: this round's groups now
#if !TC_LATE_PREFETCH
        if (r == 0 && lt + 2 < ntl) load_groups(lt + 2, 0, dst);
#endif
        uint32_t b0, b1;
        range(lt, r, b0, b1);
#ifdef TC_PROF
        const bool prof = tid == TC_EPI_WARPS * 32;
        long long c0 = clock64(), c1 = c0, c2 = c0;
#endif
        if (!TC_TMEM_A && unit >= 2) {
          mbar_wait(&empty_bar[s], ((unit >> 1) - 1u) & 1u);  // MMAs of unit - 2 done with this stage
#ifdef TC_PROF
          c1 = clock64();
#endif
          for (uint32_t e = pt; e < SLOT_B / 16; e += TC_SLOT_THREADS)
            reinterpret_cast<uint4*>(Ab)[e] = make_uint4(0u, 0u, 0u, 0u);
          asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(TC_SLOT_THREADS) : "memory");
        }
#ifdef TC_PROF
        c2 = clock64();
#endif
        if (b0 < b1) {
          const uint32_t G0 = (b0 + esh) >> 3, G1 = (b1 + esh + 7u) >> 3;
          const int lo = (int)(b0 + esh), hi = (int)(b1 + esh);  // element indices relative to the aligned base
          uint32_t* Aw = reinterpret_cast<uint32_t*>(Ab);
#pragma unroll
          for (int g = 0; g < PF; g++) {
            const uint32_t G = G0 + pt + (uint32_t)g * TC_SLOT_THREADS;
            if (G < G1) {
              // the group's photons inside [lo, hi) as a bit mask (all 8 except at the range ends)
              const int el = min(max(lo - (int)(8u * G), 0), 8), eh = min(max(hi - (int)(8u * G), 0), 8);
              const uint32_t msk = (0xffu << el) & (0xffu >> (8 - eh));
              const uint32_t w4[4] = {cur[g].x, cur[g].y, cur[g].z, cur[g].w};
#pragma unroll
              for (int e = 0; e < 8; e++) {
                const uint32_t x = (w4[e >> 1] >> ((e & 1) * 16)) & 0xffffu;
                // x < T: an out-of-range bin (precondition violation) is the zero "absent photon"
                // term (a zero increment at a wrapped in-block address)
const uint32_t inc = (((msk >> e) & 1u) & (uint32_t)(x < T)) << ((x & 1u) << 4);
                atomicAdd(Aw + ((x >> 1) & (SLOT_B / 4 - 1u)), inc);  // unconditional: a branch per photon costs more
              }
            }
          }
        }
#if TC_LATE_PREFETCH
        // tile lt + 2's groups issued only after this tile's registers were consumed: issued at the top
        // of the body they shared scoreboards with them, and the scatter waited for the new loads too
        if (r == 0 && lt + 2 < ntl) load_groups(lt + 2, 0, dst);
#endif
#if TC_TMEM_A
        {  // counts -> normal fp16 (c 2^-14, HMUL2 by 2^10) straight into TMEM A stage s: lane = row
           // a of this slot's pixel, warp wi takes 16-element K groups wi, wi + 4, ...; each 16-byte
           // chunk is zeroed as it is read (the next unit scatters into the same histogram)
          asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(TC_SLOT_THREADS) : "memory");
          if (unit >= 2) mbar_wait(&empty_bar[s], ((unit >> 1) - 1u) & 1u);  // MMAs of unit - 2 read stage s
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const __half2 s10 = __float2half2_rn(1024.f);
          const uint32_t rowb = (uint32_t)(lane >> 3) * 16u * Kb + (uint32_t)(lane & 7) * 16u;
          const uint32_t ta = tmem + ((slot * 32u) << 16) + 2u * (uint32_t)N + s * (Kb >> 1);
          for (uint32_t g = wi; g < Kb / 16u; g += TC_BLD_PER_SLOT) {
            uint32_t rr[8];
#pragma unroll
            for (int h = 0; h < 2; h++) {  // k_hi = 2 g + h
              uint4* cp = reinterpret_cast<uint4*>(Ab + rowb + (2u * g + (uint32_t)h) * 128u);
              uint4 w = *cp;
              *cp = make_uint4(0u, 0u, 0u, 0u);
              __half2* hh = reinterpret_cast<__half2*>(&w);
#pragma unroll
              for (int i = 0; i < 4; i++) hh[i] = __hmul2(hh[i], s10);
              rr[4 * h + 0] = w.x;
              rr[4 * h + 1] = w.y;
              rr[4 * h + 2] = w.z;
              rr[4 * h + 3] = w.w;
            }
            tmem_st8(ta + 8u * g, rr);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          // every chunk read and zeroed before any warp of the slot scatters the next unit
          asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(TC_SLOT_THREADS) : "memory");
        }
#elif TC_NORMAL_COUNTS
        {  // counts (bits c = c 2^-24 as fp16 subnormals) -> c 2^-14, normal fp16, by one exact
           // HMUL2 by 2^10 per pair, in place, once both warps of the slot have scattered
          asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(TC_SLOT_THREADS) : "memory");
          uint4* Av = reinterpret_cast<uint4*>(Ab);
          const __half2 s10 = __float2half2_rn(1024.f);
          for (uint32_t e = pt; e < SLOT_B / 16; e += TC_SLOT_THREADS) {
            uint4 w = Av[e];
            __half2* h = reinterpret_cast<__half2*>(&w);
#pragma unroll
            for (int i = 0; i < 4; i++) h[i] = __hmul2(h[i], s10);
            Av[e] = w;
          }
        }
#endif
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#ifdef TC_PROF
        if (prof) {
          const long long c3 = clock64();
          atomicAdd(&tc_prof[0], (unsigned long long)(c1 - c0));
          atomicAdd(&tc_prof[1], (unsigned long long)(c2 - c1));
          atomicAdd(&tc_prof[2], (unsigned long long)(c3 - c2));
          atomicAdd(&tc_prof[3], 1ull);
        }
#endif
        __syncwarp();
        if (tid == TC_EPI_WARPS * 32)
          uflags[s] = (r == 0 ? UF_FIRST : 0u) | (r + 1 == rounds ? UF_LAST : 0u) |
                      (r + 1 == rounds && lt + 1 == ntl ? UF_END : 0u) | ((lt & 1u) ? UF_TB : 0u);
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_bar[s]);
      }
    };
    uint4 q0[PF], q1[PF], q2[PF];
    if (ntl > 0) load_groups(0, 0, q0);
    if (ntl > 1) load_groups(1, 0, q1);
    for (uint32_t lt = 0; lt < ntl; lt += 3) {
      body(lt, q0, q2);
      if (lt + 1 < ntl) body(lt + 1, q1, q0);
      if (lt + 2 < ntl) body(lt + 2, q2, q1);
    }
  } else if (warp == TC_MMA_WARP) {
    // ======================= MMA issuer =======================
    if (lane == 0 && ntl > 0) {
      // D f32, A/B f16, both K-major, N, M = 128
      const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint32_t sa0 = su32(A0), sb = su32(Bs);
      uint32_t lt = 0;
      for (uint32_t unit = 0;; unit++) {
        const uint32_t s = unit & 1u;
        TCP_T0
        mbar_wait(&full_bar[s], (unit >> 1) & 1u);
        TCP_ADD(4, _tcp0);
        const uint32_t f = uflags[s];
        const uint32_t tb = (f & UF_TB) ? 1u : 0u;
#ifdef TC_PROF
        const long long _tcp1 = clock64();
#endif
        const uint32_t sa = sa0 + s * ASZ;
#if TC_CP
        // the stage into TMEM columns 256 + 128 s (after the MMAs of unit - 2 read them), the stage
        // released as soon as the copies land, then the MMAs with A in TMEM (98 vs 127 cycles each,
        // microbench/umma_rate.cu)
        const uint32_t ta = tmem + 256u + 128u * s;
        if (unit >= 2) mbar_wait(&afree_bar[s], ((unit >> 1) - 1u) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (uint32_t kk = 0; kk < Kb / 16; kk++) cp_128x256b(ta + kk * 8u, ns_desc(sa + kk * 256u, SBO));
        commit(&empty_bar[s]);
#endif
        if ((f & UF_FIRST) && lt >= 2) mbar_wait(&accempty_bar[tb], ((lt >> 1) - 1u) & 1u);
        TCP_ADD(5, _tcp1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#if TC_CP
        for (uint32_t kk = 0; kk < Kb / 16; kk++)
          mma_f16_ts(tmem + tb * (uint32_t)N, ta + kk * 8u, ns_desc(sb + kk * 256u, SBO), idesc,
                     (!(f & UF_FIRST) || kk > 0) ? 1u : 0u);
        commit(&afree_bar[s]);
#elif TC_TMEM_A
        for (uint32_t kk = 0; kk < Kb / 16; kk++)  // A: TMEM stage s, 8 columns (16 fp16) per K step
          mma_f16_ts(tmem + tb * (uint32_t)N, tmem + 2u * (uint32_t)N + s * (Kb >> 1) + kk * 8u,
                     ns_desc(sb + kk * 256u, SBO), idesc, (!(f & UF_FIRST) || kk > 0) ? 1u : 0u);
        commit(&empty_bar[s]);
#else
        for (uint32_t kk = 0; kk < Kb / 16; kk++)  // K step of 16 = two core matrices along K
          mma_f16(tmem + tb * (uint32_t)N, ns_desc(sa + kk * 256u, SBO), ns_desc(sb + kk * 256u, SBO), idesc,
                  (!(f & UF_FIRST) || kk > 0) ? 1u : 0u);
        commit(&empty_bar[s]);
#endif
        if (f & UF_LAST) {
          commit(&accfull_bar[tb]);
          lt++;
        }
        if (f & UF_END) break;
      }
    }
  } else {
    // ======================= epilogue: warp w = pixel slot w % 4, frequencies [MP/2 (w/4), MP/2 (w/4 + 1)) ====
    constexpr int NF = MP / 2;       // frequencies of this warp
    constexpr int NV = 2 * NF;       // values (re, im) reduced over the 32 rows: one per lane at MP = 32
    const uint32_t eslot = (uint32_t)warp & 3u, half = (uint32_t)warp >> 2, jj0 = half * NF;
    float2 wr[NF];  // this lane's (row a) twiddles for the warp's frequencies, held for the whole launch
#pragma unroll
    for (int jj = 0; jj < NF; jj++) wr[jj] = Ws[(jj0 + jj) * 32 + lane];
    uint32_t lt = 0;
    for (; lt < ntl; lt++) {
      const uint32_t tb = lt & 1u;
      const long long p = p0 + 4 * lt + eslot;
      const uint32_t n = so[4 * lt + eslot + 1] - so[4 * lt + eslot];
      TCP_T0
      mbar_wait(&accfull_bar[tb], (lt >> 1) & 1u);
      if (warp == 0 && lane == 0) TCP_ADD(6, _tcp0);
#ifdef TC_PROF
      const long long _tcp1 = clock64();
#endif
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tmem + tb * (uint32_t)N + ((eslot * 32u) << 16) + jj0;
      float acc[NV];
#pragma unroll
      for (int g = 0; g < NF / 8; g++) {
        float ch[8], sh[8], cl[8], sl[8];
        tmem_ld8(base + 0 * MP + 8 * g, ch);
        tmem_ld8(base + 1 * MP + 8 * g, sh);
        tmem_ld8(base + 2 * MP + 8 * g, cl);
        tmem_ld8(base + 3 * MP + 8 * g, sl);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int jj = 8 * g + k;
          const float pc = fmaf(cl[k], 0.000244140625f, ch[k]);  // hi + 2^-12 lo
          const float ps = fmaf(sl[k], 0.000244140625f, sh[k]);
          const float2 w = wr[jj];
          acc[2 * jj] = fmaf(w.x, pc, -w.y * ps);
          acc[2 * jj + 1] = fmaf(w.x, ps, w.y * pc);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty_bar[tb]);
      // reduce-scatter over the 32 rows a (lanes): lane l keeps the value indices with its bits
#pragma unroll
      for (int o = 16, h = NV / 2; o >= 1 && h >= 1; o >>= 1, h >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < h; i++) {
          const float send = up ? acc[i] : acc[i + h];
          const float keep = up ? acc[i + h] : acc[i];
          acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if constexpr (NV == 16) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
      if (warp == 0 && lane == 0) TCP_ADD(7, _tcp1);
      if (p < pend) {
        // 1 / n (fp16 integer counts) or 2^24 / n (counts as subnormal bit patterns)
        const float sc = n ? (float)((TC_NORMAL_COUNTS ? 16384.0 : 16777216.0) / (double)n) : 0.f;
        float* zp = reinterpret_cast<float*>(reinterpret_cast<float2*>(a.z) + (size_t)p * a.mstride + a.j0 + jj0);
        if constexpr (NV == 32) {
          // lane l holds value index l: frequency jj0 + l / 2, component l % 2
          if (jj0 + ((uint32_t)lane >> 1) < M) zp[lane] = acc[0] * sc;
        } else {
          // NV = 16: lanes l and l ^ 1 hold value index l / 2 (frequency jj0 + l / 4, component (l / 2) % 2)
          if (!(lane & 1) && jj0 + ((uint32_t)lane >> 2) < M) zp[lane >> 1] = acc[0] * sc;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((TC_CP || TC_TMEM_A) ? 512u : 2u * N));
}

template <int MP>
cudaError_t launch_tc_t(const SketchArgs& a, uint32_t M, cudaStream_t s, int num_sms) {
  auto fn = sketch_tc_kernel<MP>;
  static SmemAttrOnce attr;
  cudaError_t e = smem_attr_once(attr, fn, (int)sketch_tc_smem(TC_MAX_T, MP));
  if (e != cudaSuccess) return e;
  // one persistent CTA per SM (shared memory, TMEM), each a contiguous run of <= TC_TPC_MAX tiles
  // (its offsets staged in shared memory); frames beyond num_sms * TC_TPC_MAX tiles take several launches
  const long long per_launch = 4ll * TC_TPC_MAX * num_sms;
  for (long long pb = 0; pb < a.npix; pb += per_launch) {
    const long long pc = min(per_launch, a.npix - pb);
    const long long tiles = (pc + 3) / 4;
    const long long tpc = (tiles + num_sms - 1) / num_sms;
    const long long grid = (tiles + tpc - 1) / tpc;
    fn<<<(unsigned)grid, TC_THREADS_ALL, sketch_tc_smem(a.T, MP), s>>>(a, M, pb, pc, (uint32_t)tpc);
    cudaError_t e2 = cudaGetLastError();
    if (e2 != cudaSuccess) return e2;
  }
  return cudaSuccess;
}

}  // namespace

size_t sketch_tc_smem(uint32_t T, int MP) {
  const size_t Kb = (size_t)1 << tc_log2_kb(T);
  return 128 + 2 * 256 * Kb + (size_t)4 * MP * Kb * 2 + (size_t)MP * 32 * sizeof(float2) +
         sizeof(uint32_t) * (5 * (size_t)TC_TPC_MAX + 1);
}

cudaError_t launch_sketch_tc(int M, const SketchArgs& a, cudaStream_t s, int num_sms) {
  if (!tc_fits(a.T) || M < 1 || M > 32) return cudaErrorInvalidValue;
  if (M <= 16) return launch_tc_t<16>(a, (uint32_t)M, s, num_sms);
  return launch_tc_t<32>(a, (uint32_t)M, s, num_sms);
}

}  // namespace srt3d

#ifdef TC_PROF
extern "C" int srt3d_debug_tc_prof(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, srt3d::tc_prof, sizeof(srt3d::tc_prof)) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(srt3d::tc_prof, z, sizeof(z));
  }
  return 0;
}
#endif
