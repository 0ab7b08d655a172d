// NEXT-3 backprojection on the 5th-generation tensor cores (tcgen05 + TMEM).
//
//   g[i][n] = sum_{l=1..m} hhat_l ( Re z_il cos(2 pi l n / N) + Im z_il sin(2 pi l n / N) )
//
// (srt3d_backproject, reading A18; oracle/srt3d_ref.c srt3d_ref_backproject)
// is a dense contraction G = A B^T with A = [Re z, Im z] (npix x 2m) and
// B[n] = [hhat_l cos, hhat_l sin] (N x 2m): one GEMM with K = 2m <= 64.
//
// Design:
//  * fp32 accuracy from TF32 tensor cores by the 3-term split: x = x_hi + x_lo
//    with x_hi = tf32(x), x_lo = tf32(x - x_hi); A B = A_hi B_hi + A_hi B_lo +
//    A_lo B_hi (the dropped A_lo B_lo and the tf32 rounding of the lo parts are
//    ~2^-22 relative per product; the picks' tolerance is 1e-5 of sum |terms|).
//  * Half-grid symmetry: for n' = n + N/2, e^{i 2 pi l n'/N} = (-1)^l e^{i 2 pi l n/N}.
//    K is ordered [even l | odd l] (one 128-byte swizzle column each), so the
//    second half of the grid is D_2 = A_even B_even - A_odd B_odd: the same B
//    (N/2 rows) with the instruction descriptor's A-negate bit on the odd-l
//    column.  B (hi + lo, N/2 x 64 floats each, 128 KB at N = 512) is built once
//    per persistent CTA in shared memory (fp64 sincospi, exact index l n mod N)
//    and stays resident; only A streams.
//  * Per tile of 128 pixels: the 4 warps load the z rows (coalesced, one
//    complex per lane), split them into A_hi / A_lo in the canonical K-major
//    128-byte-swizzled layout, fence to the async proxy, and one thread issues
//    2 halves x 2 K-columns x 4 k-steps x 3 products = 48 tcgen05.mma
//    (kind::tf32, M = 128, N = N/2, K = 8) into a TMEM accumulator of N fp32
//    columns (lane = pixel), committed to an mbarrier.
//  * Epilogue: 16 warps; warp w reads TMEM lanes 32 (w % 4) .. (its pixels)
//    and the grid columns of split w / 4 (a quarter of the N columns), 32
//    columns per tcgen05.ld.  Backprojection stages each 32 x 32 block through
//    shared memory for row-contiguous stores; init_depths finds its split's
//    candidates (g_n > 0, g_n > g_{n-1}, g_n >= g_{n+1}, circular; the split's
//    boundary neighbours read from the adjacent chunks) in one pass over TMEM
//    (the next chunk's tcgen05.ld in flight while a chunk is scanned), keeping
//    per-chunk candidate bit masks and the candidates' values (in increasing n)
//    in shared memory; every pick round walks that list with the exclusion
//    zones of the earlier picks as per-chunk bit masks, the four splits' bests
//    are combined through shared memory — the oracle's rule and tie order
//    (largest g, then smallest n).  A thread whose list would overflow re-reads
//    TMEM in its rounds instead (same values, same order).
// Supported: N % 32 == 0, 32 <= N <= 512, m <= 32; other shapes use the CUDA-
// core kernel (init.cu).
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace srt3d {

namespace {

constexpr int TC_M = 128;          // pixels per tile (TMEM lanes)
constexpr int TC_SPLIT = 4;        // column splits of the epilogue: 4 warps per TMEM lane quarter
constexpr int TC_THREADS = TC_M * TC_SPLIT;
constexpr uint32_t A_CHUNK = TC_M * 128;  // one 128-byte swizzle column of A: 16 KB
constexpr int PICK_CAP = 12;              // candidate-list entries per thread (init_depths): 24 KB

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// canonical K-major SWIZZLE_128B operand: rows of 128 B, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);  // start address (16 B units)
  d |= (uint64_t)1 << 16;                           // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                 // stride byte offset: next 8-row atom
  d |= (uint64_t)1 << 46;                           // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
  return d;
}

// byte offset of float2 slot i (0..15) of row r in a 128-byte-swizzled K column
__device__ __forceinline__ uint32_t sw_off(uint32_t r, uint32_t i) {
  return r * 128u + ((((i >> 1) ^ (r & 7u)) & 7u) << 4) + ((i & 1u) << 3);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra TC_WAIT_%=;\n\t}" ::"r"(su32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// tcgen05.ld without the wait: the registers are valid only after tmem_wait()
// + tmem_regs_ready() (the empty asm ties every later use of r to a point after
// the wait, so the compiler cannot hoist a consumer above it)
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_regs_ready(uint32_t (&r)[32]) {
#pragma unroll
  for (int i = 0; i < 32; i++) asm volatile("" : "+r"(r[i]));
}

// bits of chunk [c0, c0 + 32) inside the linear interval [lo, hi] (lo <= hi)
__device__ __forceinline__ uint32_t interval_bits(int lo, int hi, int c0) {
  const int a = max(lo - c0, 0), b = min(hi - c0, 31);
  if (a > b) return 0u;
  return (0xffffffffu >> (31 - b)) & (0xffffffffu << a);
}

// bits of chunk c0 excluded by a pick at p: circular distance d with d*T < min_sep*N
__device__ __forceinline__ uint32_t excl_bits(int p, int D, int N, int c0) {
  if (D < 0) return 0u;
  if (2 * D + 1 >= N) return 0xffffffffu;
  const int lo = p - D, hi = p + D;
  uint32_t b = interval_bits(max(lo, 0), min(hi, N - 1), c0);
  if (lo < 0) b |= interval_bits(lo + N, N - 1, c0);
  if (hi >= N) b |= interval_bits(0, hi - N, c0);
  return b;
}

// max of 32 values and its index (ties: the smaller index), as a tree: the
// epilogue runs one warp per SM sub-partition, so a serial max chain would be
// latency-bound
__device__ __forceinline__ void tree_argmax32(const float (&x)[32], float& mx, int& im) {
  float y[16];
  int iy[16];
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const bool t = x[2 * k + 1] > x[2 * k];
    y[k] = t ? x[2 * k + 1] : x[2 * k];
    iy[k] = t ? 2 * k + 1 : 2 * k;
  }
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {
#pragma unroll
    for (int k = 0; k < w; k++) {
      const bool t = y[2 * k + 1] > y[2 * k];
      y[k] = t ? y[2 * k + 1] : y[2 * k];
      iy[k] = t ? iy[2 * k + 1] : iy[2 * k];
    }
  }
  mx = y[0];
  im = iy[0];
}

// KK: the pick count rounded up to 1, 2, 3, 4 or MAX_K (compile-time loop bounds and register arrays)
template <bool PICK, int KK>
__global__ void __launch_bounds__(TC_THREADS, 1) bp_tc_kernel(const BpArgs a) {
  extern __shared__ unsigned char tc_raw[];
  unsigned char* sm = tc_raw + ((1024u - (su32(tc_raw) & 1023u)) & 1023u);  // 1 KB aligned (swizzle atoms)
  const int N = (int)a.N, NH = N / 2, NC = N / 32;
  const uint32_t m = a.m;
  unsigned char* a_hi = sm;                          // 2 K columns x 16 KB
  unsigned char* a_lo = a_hi + 2 * A_CHUNK;
  unsigned char* b_hi = a_lo + 2 * A_CHUNK;          // 2 K columns x NH rows x 128 B
  unsigned char* b_lo = b_hi + 2 * NH * 128;
  __shared__ __align__(8) uint64_t mma_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ float xb_v[2][TC_SPLIT][TC_M];  // per-round local bests of the column splits
  __shared__ int xb_i[2][TC_SPLIT][TC_M];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, split = warp >> 2;  // TMEM lanes 32*quarter.. ; column split
  const int prow = quarter * 32 + lane;             // pixel row within the tile = TMEM lane
  // this thread's 32-column chunks [c0, c1) of the grid
  const int c0 = split * NC / TC_SPLIT, c1 = (split + 1) * NC / TC_SPLIT;

  // ---- one-time setup: B (hi, lo) for the first half grid, barrier, TMEM ----
  for (int e = tid; e < NH * 32; e += TC_THREADS) {
    const int n = e >> 5, s = e & 31;          // s: K slot pair index over both columns
    const int col = s >> 4, i = s & 15;        // column 0: even l = 2(i+1); column 1: odd l = 2i+1
    const uint32_t l = col == 0 ? 2u * (uint32_t)(i + 1) : 2u * (uint32_t)i + 1u;
    float2 hv = make_float2(0.f, 0.f), lv = hv;
    if (l <= m) {
      const uint32_t r = (l * (uint32_t)n) % (uint32_t)N;
      const int rc = 2 * (int)r > N ? (int)r - N : (int)r;  // centred index: argument in (-1, 1]
      double sn, cs;
      sincospi(2.0 * (double)rc / (double)N, &sn, &cs);
      const double h = (double)a.hh[l - 1];
      const double vc = h * cs, vs = h * sn;
      const uint32_t hc = tf32_rna((float)vc), hs = tf32_rna((float)vs);
      hv = make_float2(__uint_as_float(hc), __uint_as_float(hs));
      lv = make_float2(__uint_as_float(tf32_rna((float)(vc - (double)hv.x))),
                       __uint_as_float(tf32_rna((float)(vs - (double)hv.y))));
    }
    const uint32_t off = (uint32_t)col * (uint32_t)NH * 128u + sw_off((uint32_t)n, (uint32_t)i);
    *reinterpret_cast<float2*>(b_hi + off) = hv;
    *reinterpret_cast<float2*>(b_lo + off) = lv;
  }
  if (tid == 0) {
    mbar_init1(&mma_bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t ncols = 32;
  while ((int)ncols < N) ncols <<= 1;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  // instruction descriptors: D f32, A/B tf32, K-major, M = 128, N = NH; A negated
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NH >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
  const uint32_t idesc_neg = idesc | (1u << 13);
  const uint32_t sa_hi = su32(a_hi), sa_lo = su32(a_lo), sb_hi = su32(b_hi), sb_lo = su32(b_lo);
  const int D = a.min_sep == 0 ? -1 : (int)(((unsigned long long)a.min_sep * (unsigned)N - 1ull) / a.T);
  const float2* zg = reinterpret_cast<const float2*>(a.z);
  const long long ntiles = (a.npix + TC_M - 1) / TC_M;
  uint32_t phase = 0;

  // the z rows of a tile: warp w holds rows RPW*w .. , lane = frequency l - 1
  // (loads for tile t+1 are issued at the start of tile t's epilogue)
  constexpr int RPW = TC_M / (TC_THREADS / 32);
  float2 zpre[RPW];
  auto load_tile = [&](long long t) {
    const long long r0 = t * TC_M + warp * RPW;
#pragma unroll
    for (int rr = 0; rr < RPW; rr++) {
      const long long pix = r0 + rr;
      zpre[rr] = (t < ntiles && pix < a.npix && (uint32_t)lane < m) ? zg[(size_t)pix * m + lane] : make_float2(0.f, 0.f);
    }
  };
  load_tile(blockIdx.x);

  // ---- A staging and the MMAs of one tile (shared by both epilogues) ----
  // z rows (zpre) -> [even l | odd l] K columns, split hi / lo, swizzled
  auto stage_a = [&]() {
    const uint32_t i = (uint32_t)lane >> 1, col = (lane & 1) ? 0u : 1u;  // frequency l = lane + 1
#pragma unroll
    for (int rr = 0; rr < RPW; rr++) {
      const uint32_t r = (uint32_t)(warp * RPW + rr);
      const float2 v = zpre[rr];
      const float hx = __uint_as_float(tf32_rna(v.x)), hy = __uint_as_float(tf32_rna(v.y));
      const float lx = __uint_as_float(tf32_rna(v.x - hx)), ly = __uint_as_float(tf32_rna(v.y - hy));
      const uint32_t off = col * A_CHUNK + sw_off(r, i);
      *reinterpret_cast<float2*>(a_hi + off) = make_float2(hx, hy);
      *reinterpret_cast<float2*>(a_lo + off) = make_float2(lx, ly);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  };
  // one thread, after a CTA barrier that follows stage_a and the last TMEM reads
  auto issue_mma = [&]() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t dt = tmem + (uint32_t)(h * NH);
      int first = 1;
#pragma unroll
      for (int c = 0; c < 2; c++) {
        const uint32_t id = (h == 1 && c == 1) ? idesc_neg : idesc;
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
          const uint32_t ao = (uint32_t)c * A_CHUNK + (uint32_t)kk * 32u;
          const uint32_t bo = (uint32_t)c * (uint32_t)NH * 128u + (uint32_t)kk * 32u;
          mma_tf32(dt, sw128_desc(sa_hi + ao), sw128_desc(sb_hi + bo), id, first ? 0u : 1u);
          mma_tf32(dt, sw128_desc(sa_hi + ao), sw128_desc(sb_lo + bo), id, 1u);
          mma_tf32(dt, sw128_desc(sa_lo + ao), sw128_desc(sb_hi + bo), id, 1u);
          first = 0;
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(&mma_bar))
                 : "memory");
  };
  const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
  float v[32];

  if constexpr (!PICK) {
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const long long row0 = tile * TC_M;
      stage_a();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (tid == 0) issue_mma();
      mbar_wait_parity(&mma_bar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      load_tile(tile + gridDim.x);  // the next tile's z in flight during the epilogue
      // per 32-column chunk: the warp's 32 rows through shared memory (the A
      // buffers are free until the next tile; float4 slots XOR-swizzled) so
      // each warp store covers whole 128-byte row runs
      float* stg = reinterpret_cast<float*>(a_hi) + warp * 32 * 32;
      for (int c = c0; c < c1; c++) {
        tmem_ld32(trow + (uint32_t)(c * 32), v);
#pragma unroll
        for (int q = 0; q < 8; q++)
          *reinterpret_cast<float4*>(stg + lane * 32 + 4 * (q ^ (lane & 7))) =
              make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; q++) {  // 4 rows x 128 B per warp store
          const int r = q * 4 + (lane >> 3), c4 = lane & 7;
          const long long pr = row0 + quarter * 32 + r;
          if (pr < a.npix)
            *reinterpret_cast<float4*>(a.g + (size_t)pr * N + c * 32 + 4 * c4) =
                *reinterpret_cast<const float4*>(stg + r * 32 + 4 * (c4 ^ (r & 7)));
        }
        __syncwarp();
      }
      // the next tile's MMAs overwrite the accumulator and A: all reads done first
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
    }
  } else {
    // init_depths, pipelined across tiles: tile t+1's z loads overlap tile t's
    // MMAs; A(t+1) is staged as soon as MMA(t) has completed; the TMEM scan of
    // tile t leaves every candidate in shared memory (masks in registers,
    // values in the list), so MMA(t+1) is issued right after the scan and runs
    // under tile t's pick rounds (unless some thread's list overflowed: then
    // the rounds re-read TMEM and MMA(t+1) waits for them).
    constexpr int MAXC = 16 / TC_SPLIT;  // chunks per split (N <= 512)
    float* const lst = reinterpret_cast<float*>(b_lo + 2 * NH * 128) + tid;  // entry e at lst[e * TC_THREADS]
    float* const lend = lst + a.list_cap * TC_THREADS;
    long long tile = blockIdx.x;
    if (tile < ntiles) {
      stage_a();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (tid == 0) issue_mma();
    }
    for (; tile < ntiles; tile += gridDim.x) {
      const long long row0 = tile * TC_M, nxt = tile + gridDim.x;
      const bool has_next = nxt < ntiles;
      load_tile(nxt);
      mbar_wait_parity(&mma_bar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (has_next) stage_a();  // MMA(t) has read A
      const long long pix = row0 + prow;

      // ---- TMEM scan: candidate masks (registers) and values (list) ----
      // candidate: g_n > 0, g_n > g_{n-1}, g_n >= g_{n+1} (circular); values
      // appended in increasing n while the list has room; a thread with more
      // than PICK_CAP candidates (measured at C5: at most 9 of 128 columns) is
      // marked overflowed
      uint32_t cbm[MAXC];
#pragma unroll
      for (int i = 0; i < MAXC; i++) cbm[i] = 0u;
      float* wp = lst;
      if (c1 > c0) {
        uint32_t ra[32], rb[32];
        tmem_ld32_async(trow + (uint32_t)(((c0 + NC - 1) % NC) * 32), ra);
        tmem_ld32_async(trow + (uint32_t)((c1 % NC) * 32), rb);
        tmem_wait();
        tmem_regs_ready(ra);
        tmem_regs_ready(rb);
        float prevv = __uint_as_float(ra[31]);       // g[32 c0 - 1] (circular)
        const float nextv = __uint_as_float(rb[0]);  // g[32 c1] (circular)
        float pend = 0.f, pendp = 0.f;
        tmem_ld32_async(trow + (uint32_t)(c0 * 32), ra);
        tmem_wait();
        tmem_regs_ready(ra);
        auto chunk = [&](uint32_t(&r)[32], uint32_t(&rn)[32], int i) {
          const int c = c0 + i;
          if (c + 1 < c1) tmem_ld32_async(trow + (uint32_t)((c + 1) * 32), rn);  // in flight during the scan
          const float v0 = __uint_as_float(r[0]);
          if (i > 0) {  // element 31 of chunk c-1 (its right neighbour is v[0])
            const bool ok = pend > 0.f && pend > pendp && pend >= v0;
            if (ok) cbm[i - 1] |= 1u << 31;
            if (ok && wp < lend) {
              *wp = pend;
              wp += TC_THREADS;
            }
          }
          uint32_t bits = 0u;
#pragma unroll
          for (int e = 0; e < 31; e++) {
            const float g = __uint_as_float(r[e]), gp = e == 0 ? prevv : __uint_as_float(r[e - 1]);
            const bool ok = g > 0.f && g > gp && g >= __uint_as_float(r[e + 1]);
            if (ok) bits |= 1u << e;
            if (ok && wp < lend) {
              *wp = g;
              wp += TC_THREADS;
            }
          }
          cbm[i] = bits;
          pend = __uint_as_float(r[31]);
          pendp = __uint_as_float(r[30]);
          prevv = pend;
          if (c + 1 < c1) {
            tmem_wait();
            tmem_regs_ready(rn);
          }
        };
#pragma unroll
        for (int i = 0; i < MAXC; i++) {
          if (c0 + i >= c1) break;
          if (i & 1)
            chunk(rb, ra, i);
          else
            chunk(ra, rb, i);
        }
        const bool ok = pend > 0.f && pend > pendp && pend >= nextv;  // n = 32 c1 - 1
#pragma unroll
        for (int i = 0; i < MAXC; i++)
          if (ok && i == c1 - c0 - 1) cbm[i] |= 1u << 31;
        if (ok && wp < lend) *wp = pend;
      }
      int ncand = 0, pos0[MAXC];
#pragma unroll
      for (int i = 0; i < MAXC; i++) {
        pos0[i] = ncand;
        ncand += __popc(cbm[i]);
      }
      const bool ovf = ncand > a.list_cap;
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      const bool any_ovf = __syncthreads_or(ovf) != 0;  // also: A(t+1) staged by every warp
      if (has_next && !any_ovf && tid == 0) issue_mma();  // runs under the pick rounds
      const bool wovf = __any_sync(0xffffffffu, ovf);

      // ---- K rounds: each split's best outside the exclusion zones of the
      // picks so far, combined across the splits (largest g, then smallest n);
      // every split thread of a pixel keeps the same pick list ----
      uint32_t el[MAXC];
#pragma unroll
      for (int i = 0; i < MAXC; i++) el[i] = cbm[i];
      int pick[KK];
      float pg[KK];
      int cnt = 0, lastp = 0;
      for (uint32_t k = 0; k < a.K; k++) {
        const int buf = k & 1;
        float best = 0.f;
        int bn = -1;
        const bool live = cnt == (int)k;
        if (k > 0 && live) {  // narrowed by the newest pick's exclusion zone
#pragma unroll
          for (int i = 0; i < MAXC; i++) el[i] &= ~excl_bits(lastp, D, N, (c0 + i) * 32);
        }
        if (live && !ovf) {
#pragma unroll
          for (int i = 0; i < MAXC; i++) {
            uint32_t e = el[i];
            while (e) {  // increasing n: strict > keeps the smaller n
              const int j = __ffs(e) - 1;
              e &= e - 1u;
              const float val = lst[(pos0[i] + __popc(cbm[i] & ((1u << j) - 1u))) * TC_THREADS];
              if (val > best) {
                best = val;
                bn = (c0 + i) * 32 + j;
              }
            }
          }
        }
        if (wovf) {  // warp-uniform: TMEM re-reads for the overflowed lanes (MMA(t+1) not issued yet)
#pragma unroll
          for (int i = 0; i < MAXC; i++) {
            if (c0 + i >= c1) break;
            const uint32_t elig = live && ovf ? el[i] : 0u;
            if (!__any_sync(0xffffffffu, elig != 0u)) continue;
            tmem_ld32(trow + (uint32_t)((c0 + i) * 32), v);
#pragma unroll
            for (int q = 0; q < 32; q++) v[q] = ((elig >> q) & 1u) ? v[q] : 0.f;
            float cm;
            int ci;
            tree_argmax32(v, cm, ci);
            if (cm > best) {
              best = cm;
              bn = (c0 + i) * 32 + ci;
            }
          }
        }
        xb_v[buf][split][prow] = best;
        xb_i[buf][split][prow] = bn;
        // a pixel's four split threads sit in the four warps of its TMEM lane
        // quarter: a named barrier over those 128 threads (not the CTA) joins them
        asm volatile("bar.sync %0, %1;" ::"r"(1 + quarter), "r"(4 * 32) : "memory");
        float gb = 0.f;
        int gi = -1;
#pragma unroll
        for (int q = 0; q < TC_SPLIT; q++) {  // splits cover increasing n: strict > keeps the smaller n
          const int qi = xb_i[buf][q][prow];
          const float qv = xb_v[buf][q][prow];
          if (qi >= 0 && (gi < 0 || qv > gb)) {
            gb = qv;
            gi = qi;
          }
        }
        if (cnt == (int)k && gi >= 0) {
#pragma unroll
          for (int q = 0; q < KK; q++)
            if (q == cnt) {
              pick[q] = gi;
              pg[q] = gb;
            }
          lastp = gi;
          cnt++;
        }
      }
      if (pix < a.npix) {
        // sort by depth (insertion sort on the register arrays: compile-time
        // indices); the four split threads of a pixel write every 4th pick
#pragma unroll
        for (int x = 1; x < KK; x++)
#pragma unroll
          for (int y = x; y > 0; y--)
            if (y < cnt && pick[y - 1] > pick[y]) {
              const int tp = pick[y];
              pick[y] = pick[y - 1];
              pick[y - 1] = tp;
              const float tg = pg[y];
              pg[y] = pg[y - 1];
              pg[y - 1] = tg;
            }
#pragma unroll
        for (int k = 0; k < KK; k++) {
          if (k >= (int)a.K) break;
          if ((k & (TC_SPLIT - 1)) != split) continue;
          const size_t o = (size_t)pix * a.K + k;
          if (k < cnt) {
            a.t_out[o] = (float)((double)pick[k] * (double)a.T / (double)N);
            a.g_out[o] = pg[k];
            a.a_out[o] = fminf(fmaxf(pg[k] * a.inv_sh2, 0.f), 1.f);
          } else {
            const double tfirst = cnt ? (double)pick[0] * (double)a.T / (double)N : 0.0;
            a.t_out[o] = (float)fmod(tfirst + 0.5 * (double)a.T, (double)a.T);
            a.g_out[o] = 0.f;
            a.a_out[o] = 0.f;
          }
        }
        if (split == TC_SPLIT - 1) a.count[pix] = cnt;
      }
      if (has_next && any_ovf) {  // the rounds' TMEM reads are done
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (tid == 0) issue_mma();
      }
      __syncthreads();  // the next scan rewrites the lists and the combine buffers
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

size_t bp_tc_smem(uint32_t N, bool pick) {
  const size_t nh = N / 2;
  return 1024 + 4 * (size_t)A_CHUNK + 2 * 2 * nh * 128 + (pick ? sizeof(float) * PICK_CAP * TC_THREADS : 0);
}

}  // namespace

bool backproject_tc_supported(uint32_t N, uint32_t m) { return m <= 32 && N % 32 == 0 && N >= 32 && N <= 512; }

cudaError_t launch_backproject_tc(const BpArgs& a, bool pick, cudaStream_t s, int num_sms) {
  if (a.npix <= 0) return cudaSuccess;
  const int kk = !pick ? 1 : a.K <= 1 ? 1 : a.K == 2 ? 2 : a.K == 3 ? 3 : a.K == 4 ? 4 : MAX_K;
  const int vi = !pick ? 0 : kk == 1 ? 1 : kk == 2 ? 2 : kk == 3 ? 3 : kk == 4 ? 4 : 5;
  void (*const fns[6])(const BpArgs) = {bp_tc_kernel<false, 1>, bp_tc_kernel<true, 1>, bp_tc_kernel<true, 2>,
                                        bp_tc_kernel<true, 3>,  bp_tc_kernel<true, 4>, bp_tc_kernel<true, MAX_K>};
  auto fn = fns[vi];
  static SmemAttrOnce attr[6];
  cudaError_t e = smem_attr_once(attr[vi], fn, (int)bp_tc_smem(512, pick));
  if (e != cudaSuccess) return e;
  // SRT3D_INIT_LIST_CAP (tests only) shrinks the candidate list so that the
  // overflow path (TMEM re-reads, MMA of the next tile after the rounds) runs
  BpArgs b = a;
  b.list_cap = PICK_CAP;
  if (const char* e = getenv("SRT3D_INIT_LIST_CAP")) b.list_cap = max(0, min(PICK_CAP, atoi(e)));
  const long long tiles = (a.npix + TC_M - 1) / TC_M;
  long long grid = num_sms;  // one persistent CTA per SM (the accumulator holds up to all 512 TMEM columns)
  if (grid > tiles) grid = tiles;
  fn<<<(unsigned)grid, TC_THREADS, bp_tc_smem(a.N, pick), s>>>(b);
  return cudaGetLastError();
}

}  // namespace srt3d
