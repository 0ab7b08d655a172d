// NEXT-4 — streaming acquisition: the sketch "can be updated
// in an online fashion with each incoming photon".
//
//   srt3d_sketch_merge: z = (n_a z_a + n_b z_b) / (n_a + n_b), n = n_a + n_b
//      — folds the sketch of a new photon batch into a running
//     sketch; in place (z_out = z_a, n_out = n_a) is allowed.
//   srt3d_bucket_events: an unsorted (pixel, bin) event stream -> the
//     pixel-sorted CSR frame srt3d_sketch consumes (reading A21), as a
//     two-level counting sort whose writes are coalesced:
//       A. per chunk of 32768 events, a shared-memory histogram of the coarse
//          key (pixel >> S, <= 512 buckets) -> table[bucket][chunk];
//       scan of the table (bucket-major) -> the segment of every
//          (bucket, chunk) in a packed temp buffer;
//       B. the chunk again, in tiles of 8192 events stably sorted by bucket
//          in shared memory (stable_rank below), written to the segments
//          packed as (pixel & (2^S - 1)) << 16 | bin;
//       C. one CTA per bucket: histogram of the local pixel -> exact per-pixel
//          offsets; then tiles of 8192 events stably sorted by local pixel
//          and written out in pixel order (runs of consecutive addresses
//          instead of one random 2-byte store per event).
//     Every stage preserves stream order, so the result is the stable sort by
//     pixel: deterministic, bit-identical to the oracle's counting sort
//     (SURVEY §4 T7).  Frames with more than 512 * 8192 pixels use a one-level
//     variant (global atomic counts, scan, atomic scatter: within-pixel order
//     follows atomic arrival).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace srt3d {

// One warp per pixel, four pixels per warp iteration with every load issued
// before any arithmetic (the counts, then the 2 x 4 rows: for m = 32 eight 8-byte
// loads in flight per lane); counts are read before the (possibly aliased) count
// output is written; the row's m complex values are spread over the lanes.
// nb == nullptr: n_b[i] = offs_b[i+1] - offs_b[i] (the batch's CSR offsets).
constexpr int MERGE_U = 4;
__global__ void __launch_bounds__(256) merge_kernel(const float2* __restrict__ za, const uint32_t* na,
                                                    const float2* __restrict__ zb, const uint32_t* nb,
                                                    const uint32_t* offs_b, long long npix, uint32_t m, float2* zo,
                                                    uint32_t* no) {
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * MERGE_U; i0 < npix;
       i0 += nw * MERGE_U) {
    uint32_t ca[MERGE_U], cb[MERGE_U];
#pragma unroll
    for (int u = 0; u < MERGE_U; u++) {
      const long long i = i0 + u;
      ca[u] = i < npix ? na[i] : 0u;
      cb[u] = i < npix ? (nb ? nb[i] : offs_b[i + 1] - offs_b[i]) : 0u;
    }
    for (uint32_t j0 = 0; j0 < m; j0 += 32) {
      const uint32_t j = j0 + lane;
      float2 x[MERGE_U], y[MERGE_U];
#pragma unroll
      for (int u = 0; u < MERGE_U; u++) {
        const long long i = i0 + u;
        const bool ok = i < npix && j < m;
        x[u] = ok ? za[(size_t)i * m + j] : make_float2(0.f, 0.f);
        y[u] = ok ? zb[(size_t)i * m + j] : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < MERGE_U; u++) {
        const long long i = i0 + u;
        if (i >= npix || j >= m) continue;
        const uint64_t n = (uint64_t)ca[u] + cb[u];
        const double inv = n ? 1.0 / (double)n : 0.0;
        const float wa = (float)((double)ca[u] * inv), wb = (float)((double)cb[u] * inv);
        zo[(size_t)i * m + j] = make_float2(fmaf(wa, x[u].x, wb * y[u].x), fmaf(wa, x[u].y, wb * y[u].y));
      }
    }
    __syncwarp();
    uint32_t nsum = 0u;
#pragma unroll
    for (int u = 0; u < MERGE_U; u++)
      if (lane == u) nsum = ca[u] + cb[u];
    if (lane < MERGE_U && i0 + lane < npix) no[i0 + lane] = nsum;
  }
}

// Even m with 16-byte-aligned rows (C5): a warp merges blocks of 8 pixels
// (8 m complex = 4 m float4, contiguous in all three arrays) with 16-byte loads,
// consecutive lanes on consecutive addresses; lanes 0..7 read the block's
// counts first, form the weights in fp64 exactly as merge_kernel does (one
// rounding each), and hand them to the other lanes by shuffle; every load of
// the block is issued before any arithmetic.  A block's pixels are touched by
// this warp only, so in-place accumulation stays safe.
constexpr int MERGE_BP = 8;             // pixels per block
// V: float4 per lane per block (m <= 8 V)
template <int MERGE_V>
__global__ void __launch_bounds__(256) merge_kernel_v4(const float4* __restrict__ za, const uint32_t* na,
                                                       const float4* __restrict__ zb, const uint32_t* nb,
                                                       const uint32_t* offs_b, long long npix, uint32_t m, float4* zo,
                                                       uint32_t* no) {
  const int lane = threadIdx.x & 31;
  const uint32_t h = m / 2;  // float4 per row
  const uint32_t nv = MERGE_BP * h;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * MERGE_BP; i0 < npix;
       i0 += nw * MERGE_BP) {
    const long long ip = i0 + lane;
    uint32_t ca = 0u, cb = 0u;
    if (lane < MERGE_BP && ip < npix) {
      ca = na[ip];
      cb = nb ? nb[ip] : offs_b[ip + 1] - offs_b[ip];
    }
    const long long e0 = i0 * h;
    const long long eend = npix * (long long)h;
    float4 x[MERGE_V], y[MERGE_V];
#pragma unroll
    for (int q = 0; q < MERGE_V; q++) {
      const uint32_t e = (uint32_t)lane + 32u * q;
      const bool ok = e < nv && e0 + e < eend;
      x[q] = ok ? za[e0 + e] : make_float4(0.f, 0.f, 0.f, 0.f);
      y[q] = ok ? zb[e0 + e] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const uint64_t n = (uint64_t)ca + cb;
    const double inv = n ? 1.0 / (double)n : 0.0;
    const float wa_l = (float)((double)ca * inv), wb_l = (float)((double)cb * inv);
#pragma unroll
    for (int q = 0; q < MERGE_V; q++) {
      const uint32_t e = (uint32_t)lane + 32u * q;
      const int src = (int)(min(e, nv - 1u) / h);  // the element's pixel within the block
      const float wa = __shfl_sync(0xffffffffu, wa_l, src), wb = __shfl_sync(0xffffffffu, wb_l, src);
      if (e < nv && e0 + e < eend)
        zo[e0 + e] = make_float4(fmaf(wa, x[q].x, wb * y[q].x), fmaf(wa, x[q].y, wb * y[q].y),
                                 fmaf(wa, x[q].z, wb * y[q].z), fmaf(wa, x[q].w, wb * y[q].w));
    }
    if (lane < MERGE_BP && ip < npix) no[ip] = ca + cb;
  }
}

cudaError_t launch_merge(const float* za, const uint32_t* na, const float* zb, const uint32_t* nb,
                         const uint32_t* offs_b, long long npix, uint32_t m, float* zo, uint32_t* no, cudaStream_t s,
                         int num_sms) {
  if (npix <= 0) return cudaSuccess;
  const bool v4 = m % 2 == 0 && m <= MAX_M && (((uintptr_t)za | (uintptr_t)zb | (uintptr_t)zo) & 15u) == 0;
  if (v4) {
    long long grid = (npix + 8 * MERGE_BP - 1) / (8 * MERGE_BP);
    if (grid > (long long)num_sms * 8) grid = (long long)num_sms * 8;
    auto fn = m <= 32 ? merge_kernel_v4<4> : merge_kernel_v4<MAX_M / 8>;
    fn<<<(unsigned)grid, 256, 0, s>>>(reinterpret_cast<const float4*>(za), na, reinterpret_cast<const float4*>(zb),
                                      nb, offs_b, npix, m, reinterpret_cast<float4*>(zo), no);
    return cudaGetLastError();
  }
  long long grid = (npix + 8 * MERGE_U - 1) / (8 * MERGE_U);
  if (grid > (long long)num_sms * 8) grid = (long long)num_sms * 8;
  merge_kernel<<<(unsigned)grid, 256, 0, s>>>(reinterpret_cast<const float2*>(za), na,
                                              reinterpret_cast<const float2*>(zb), nb, offs_b, npix, m,
                                              reinterpret_cast<float2*>(zo), no);
  return cudaGetLastError();
}

// ---- bucketing --------------------------------------------------------------
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_PER_THREAD = 4;
constexpr long long SCAN_TILE = (long long)SCAN_THREADS * SCAN_PER_THREAD;

constexpr int BK_CHUNK = 32768;     // events per CTA in passes A and B
constexpr int BK_MAX_BUCKETS = 512;  // coarse buckets
constexpr int BK_MAX_S = 13;         // log2 pixels per bucket (local pixel id in 16 bits, smem histograms)
constexpr int BK_TILE = 8192;        // events per shared-memory sorted tile (passes B, C)

static int bucket_shift(long long npix) {
  int S = 0;
  while ((npix + (1ll << S) - 1) >> S > BK_MAX_BUCKETS) S++;
  return S;
}
static bool bucket_two_level(long long npix) { return npix > 0 && bucket_shift(npix) <= BK_MAX_S; }

size_t bucket_scratch_words(long long npix, unsigned long long nev) {
  if (!bucket_two_level(npix)) {
    const long long nb = (npix + SCAN_TILE - 1) / SCAN_TILE;
    return (size_t)npix + (size_t)nb + 2;  // counts/cursors, block sums, dropped, total
  }
  const int S = bucket_shift(npix);
  const long long NB = (npix + (1ll << S) - 1) >> S;
  const long long nch = ((long long)nev + BK_CHUNK - 1) / BK_CHUNK;
  const long long tn = NB * (nch > 0 ? nch : 1) + 1;
  // temp, table (+ total), scan block sums, dropped, total
  return (size_t)nev + (size_t)tn + (size_t)((tn + SCAN_TILE - 1) / SCAN_TILE) + 2;
}

__global__ void count_kernel(const uint32_t* __restrict__ pix, unsigned long long nev, long long npix,
                             uint32_t* cnt, uint32_t* dropped) {
  const unsigned long long nt = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t drop = 0;
  for (unsigned long long e0 = t0; e0 < nev; e0 += 4 * nt) {
    uint32_t p[4];
    bool in[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const unsigned long long e = e0 + q * nt;
      in[q] = e < nev;
      p[q] = in[q] ? __ldcs(pix + e) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      if (!in[q]) continue;
      if ((long long)p[q] < npix)
        atomicAdd(cnt + p[q], 1u);
      else
        drop++;
    }
  }
  if (drop) atomicAdd(dropped, drop);
}

// Block-local exclusive scan of a SCAN_TILE slice of cnt into offsets; block total to bsum.
__global__ void __launch_bounds__(SCAN_THREADS) scan_tiles_kernel(const uint32_t* cnt, long long npix,
                                                                   uint32_t* offsets, uint32_t* bsum) {
  __shared__ uint32_t wsum[SCAN_THREADS / 32];
  const long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_PER_THREAD;
  uint32_t v[SCAN_PER_THREAD];
  uint32_t tsum = 0;
#pragma unroll
  for (int q = 0; q < SCAN_PER_THREAD; q++) {
    v[q] = base + q < npix ? cnt[base + q] : 0u;
    tsum += v[q];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    wsum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  uint32_t run = x - tsum + (warp ? wsum[warp - 1] : 0u);  // exclusive prefix of this thread
#pragma unroll
  for (int q = 0; q < SCAN_PER_THREAD; q++) {
    if (base + q < npix) offsets[base + q] = run;
    run += v[q];
  }
  if (threadIdx.x == SCAN_THREADS - 1) bsum[blockIdx.x] = run;  // block total
}

// Exclusive scan of the block sums (one block, sequential chunks of 1024).
__global__ void __launch_bounds__(SCAN_THREADS) scan_bsum_kernel(uint32_t* bsum, long long nb, uint32_t* total) {
  __shared__ uint32_t wsum[SCAN_THREADS / 32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (long long c0 = 0; c0 < nb; c0 += SCAN_THREADS) {
    const long long i = c0 + threadIdx.x;
    const uint32_t v = i < nb ? bsum[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const uint32_t incl = x + (warp ? wsum[warp - 1] : 0u);
    if (i < nb) bsum[i] = carry + incl - v;
    __syncthreads();
    if (threadIdx.x == SCAN_THREADS - 1) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// offsets += block prefix; cursors = offsets; offsets[npix] = total.
__global__ void scan_fix_kernel(uint32_t* offsets, uint32_t* cursor, const uint32_t* bsum, long long npix,
                                const uint32_t* total) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= npix; i += stride) {
    if (i == npix) {
      offsets[npix] = *total;
      continue;
    }
    const uint32_t o = offsets[i] + bsum[i / SCAN_TILE];
    offsets[i] = o;
    cursor[i] = o;
  }
}

// 4 events per thread per iteration: four independent atomics in flight.
__global__ void scatter_kernel(const uint32_t* __restrict__ pix, const uint16_t* __restrict__ bins,
                               unsigned long long nev, long long npix, uint32_t* cursor, uint16_t* out) {
  const unsigned long long nt = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (unsigned long long e0 = t0; e0 < nev; e0 += 4 * nt) {
    uint32_t p[4];
    uint16_t b[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const unsigned long long e = e0 + q * nt;
      p[q] = e < nev ? __ldcs(pix + e) : 0xffffffffu;
      b[q] = e < nev ? __ldcs(bins + e) : (uint16_t)0;
    }
    uint32_t pos[4];
#pragma unroll
    for (int q = 0; q < 4; q++)
      if ((long long)p[q] < npix) pos[q] = atomicAdd(cursor + p[q], 1u);
#pragma unroll
    for (int q = 0; q < 4; q++)
      if ((long long)p[q] < npix) out[pos[q]] = b[q];
  }
}

// ---- two-level bucketing ------------------------------------------------------
// In-place exclusive scan helpers over n words: scan_tiles_kernel (block
// prefix + block sums), scan_bsum_kernel, then add the block prefix.
__global__ void scan_add_kernel(uint32_t* a, const uint32_t* bsum, long long n, const uint32_t* total) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += stride)
    a[i] = i == n ? *total : a[i] + bsum[i / SCAN_TILE];
}

// Pass A: coarse histogram of one chunk -> table[b * nch + chunk].
__global__ void __launch_bounds__(512) coarse_count_kernel(const uint32_t* __restrict__ pix, unsigned long long nev,
                                                           long long npix, int S, int NB, long long nch,
                                                           uint32_t* table, uint32_t* dropped) {
  __shared__ uint32_t h[BK_MAX_BUCKETS];
  for (int b = threadIdx.x; b < NB; b += blockDim.x) h[b] = 0u;
  __syncthreads();
  const unsigned long long c0 = (unsigned long long)blockIdx.x * BK_CHUNK;
  const unsigned long long c1 = min(nev, c0 + BK_CHUNK);
  uint32_t drop = 0;
  auto count = [&](uint32_t p) {
    if ((long long)p < npix)
      atomicAdd(&h[p >> S], 1u);
    else
      drop++;
  };
  // 16-byte loads (four events each, four in flight per thread) over the chunk's aligned body
  // (chunks start at multiples of 4 events: a 16-byte-aligned pix makes every chunk aligned);
  // the scalar loop takes the chunk's last < 4 events, or everything if pix is misaligned
  unsigned long long v1 = c0;
  if ((reinterpret_cast<uintptr_t>(pix) & 15u) == 0) {
    const uint4* pv = reinterpret_cast<const uint4*>(pix + c0);
    const unsigned long long nv = (c1 - c0) >> 2;
    for (unsigned long long i0 = threadIdx.x; i0 < nv; i0 += 4ull * blockDim.x) {
      uint4 w[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const unsigned long long i = i0 + (unsigned long long)q * blockDim.x;
        w[q] = i < nv ? __ldcs(pv + i) : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      }
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (i0 + (unsigned long long)q * blockDim.x >= nv) break;
        count(w[q].x);
        count(w[q].y);
        count(w[q].z);
        count(w[q].w);
      }
    }
    v1 = c0 + 4 * nv;
  }
  for (unsigned long long e = v1 + threadIdx.x; e < c1; e += blockDim.x) count(__ldcs(pix + e));
  __syncthreads();
  for (int b = threadIdx.x; b < NB; b += blockDim.x) table[(long long)b * nch + blockIdx.x] = h[b];
  if (drop) atomicAdd(dropped, drop);
}

// Exclusive block scan of n <= 8192 shared words: out[i] = sum_{k<i} a[k]
// (out may alias a); returns the total.
__device__ uint32_t block_scan_smem(uint32_t* a, uint32_t* out, int n, uint32_t* wsum) {
  const int per = (n + blockDim.x - 1) / blockDim.x;  // contiguous run per thread
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  uint32_t t = 0;
  for (int i = lo; i < hi; i++) t += a[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = t;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t w = lane < nw ? wsum[lane] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < nw) wsum[lane] = w;
  }
  __syncthreads();
  uint32_t run = x - t + (warp ? wsum[warp - 1] : 0u);
  const uint32_t total = wsum[(blockDim.x >> 5) - 1];
  for (int i = lo; i < hi; i++) {
    const uint32_t v = a[i];
    out[i] = run;
    run += v;
  }
  __syncthreads();
  return total;
}

// ---- deterministic (stable) ranking of a tile by key ---------------------------
// The tile's events are held by the 1024-thread CTA in position order: warp w
// owns positions [256 w, 256 w + 256) as BK_ROWS rows of 32, lane l of row q at
// 256 w + 32 q + l.  Stable counting sort by key < nkeys (kbits bits):
//   1. per row, the mask of the lanes sharing the key: each lane ORs its bit
//      into a warp-private word of its key (atomicOr: the value is
//      order-independent, so deterministic — unlike ranks taken from atomic
//      arrival; 2.4x faster than ballots over the key bits and 5.7x faster than
//      __match_any_sync on sm_100a, microbench/match_vs_ballot.cu), and a
//      warp-private running count per key,
//      cnt[k * 32 + w], gives each event its rank among the warp's events of
//      that key (stored at cnt[k * 33 + w]: the pad word makes the 32 lanes'
//      different keys fall in different banks);
//   2. an exclusive scan of cnt in key-major, warp-minor order (the pad words
//      are zero) gives the first position of (key k, warp w);
//   3. position = scan + rank.
// Output positions pos[q] for the valid events (bit q of vmask); the scanned
// cnt stays in shared memory (cnt[k * 33] = first position of key k; the caller
// syncs before reusing cnt).  Returns the number of valid events.
constexpr int BK_ROWS = BK_TILE / 1024;  // 8 rows of 32 per warp
// pm: [32][nkeys] warp-private peer-mask words.
__device__ __forceinline__ uint32_t stable_rank(const uint32_t (&key)[BK_ROWS], uint32_t vmask,
                                                uint32_t (&pos)[BK_ROWS], uint32_t* cnt, uint32_t* pm, int nkeys,
                                                uint32_t* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < nkeys * 33; i += blockDim.x) cnt[i] = 0u;
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t* mw = pm + warp * nkeys;
#pragma unroll
  for (int q = 0; q < BK_ROWS; q++) {
    const bool v = (vmask >> q) & 1u;
    const uint32_t k = v ? key[q] : 0u;
    if (v) mw[k] = 0u;
    __syncwarp();
    if (v) atomicOr(&mw[k], 1u << lane);
    __syncwarp();
    const uint32_t peers = v ? mw[k] : 0u;
    uint32_t* c = cnt + k * 33u + warp;
    const uint32_t cur = *c;
    __syncwarp();
    if (v && (peers & lt) == 0u) *c = cur + __popc(peers);  // the first lane of the key's group
    __syncwarp();
    pos[q] = cur + __popc(peers & lt);
  }
  __syncthreads();
  const uint32_t total = block_scan_smem(cnt, cnt, nkeys * 33, wsum);
#pragma unroll
  for (int q = 0; q < BK_ROWS; q++)
    if ((vmask >> q) & 1u) pos[q] += cnt[key[q] * 33u + warp];
  return total;
}

// Pass B: the chunk again, in tiles of BK_TILE events stably sorted by bucket
// in shared memory (stable_rank), then written out in bucket order:
// consecutive threads store consecutive addresses of a (bucket, chunk)
// segment, and each segment keeps the events' stream order.
__global__ void __launch_bounds__(1024) partition_kernel(const uint32_t* __restrict__ pix,
                                                         const uint16_t* __restrict__ bins, unsigned long long nev,
                                                         long long npix, int S, int NB, long long nch,
                                                         const uint32_t* table, uint32_t* temp) {
  __shared__ uint32_t cur[BK_MAX_BUCKETS], wsum[32];
  extern __shared__ uint32_t pt_smem[];
  uint32_t* cnt = pt_smem;                                              // [NB * 33] stable-rank counters
  uint32_t* pm = cnt + BK_MAX_BUCKETS * 33;                             // [32][NB] peer masks
  uint32_t* sbuf = pm + BK_MAX_BUCKETS * 32;                            // [BK_TILE] packed values
  uint16_t* skey = reinterpret_cast<uint16_t*>(sbuf + BK_TILE);         // [BK_TILE] bucket
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = threadIdx.x; b < NB; b += blockDim.x) cur[b] = table[(long long)b * nch + blockIdx.x];
  const unsigned long long c0 = (unsigned long long)blockIdx.x * BK_CHUNK;
  const unsigned long long c1 = min(nev, c0 + BK_CHUNK);
  const uint32_t mask = (1u << S) - 1u;
  // this thread's events of a tile: positions 256 warp + 32 q + lane; the next
  // tile's events are loaded while the current one is sorted and written
  uint32_t np[BK_ROWS], nb[BK_ROWS];
#pragma unroll
  for (int q = 0; q < BK_ROWS; q++) {
    const unsigned long long e = c0 + 256 * warp + 32 * q + lane;
    np[q] = e < c1 ? __ldcs(pix + e) : 0xffffffffu;
    nb[q] = e < c1 ? (uint32_t)__ldcs(bins + e) : 0u;
  }
  for (unsigned long long t0 = c0; t0 < c1; t0 += BK_TILE) {
    uint32_t key[BK_ROWS], val[BK_ROWS], pos[BK_ROWS];
    uint32_t vm = 0;
#pragma unroll
    for (int q = 0; q < BK_ROWS; q++) {
      const uint32_t p = np[q];
      const bool v = (long long)p < npix;  // events past the chunk end carry 0xffffffff
      vm |= (uint32_t)v << q;
      key[q] = v ? (p >> S) : 0u;
      val[q] = nb[q] | ((p & mask) << 16);
    }
#pragma unroll
    for (int q = 0; q < BK_ROWS; q++) {
      const unsigned long long e = t0 + BK_TILE + 256 * warp + 32 * q + lane;
      np[q] = e < c1 ? __ldcs(pix + e) : 0xffffffffu;
      nb[q] = e < c1 ? (uint32_t)__ldcs(bins + e) : 0u;
    }
    const uint32_t nt = stable_rank(key, vm, pos, cnt, pm, NB, wsum);
#pragma unroll
    for (int q = 0; q < BK_ROWS; q++)
      if ((vm >> q) & 1u) {
        sbuf[pos[q]] = val[q];
        skey[pos[q]] = (uint16_t)key[q];
      }
    __syncthreads();
    for (int i = threadIdx.x; i < (int)nt; i += blockDim.x) {
      const uint32_t b = skey[i];
      temp[cur[b] + i - cnt[b * 33]] = sbuf[i];  // cnt[b * 33]: first tile position of bucket b
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NB; b += blockDim.x)
      cur[b] += (b + 1 < NB ? cnt[(b + 1) * 33] : nt) - cnt[b * 33];
    __syncthreads();
  }
}

// Pass C: one CTA per bucket — per-pixel offsets from a histogram of the
// bucket (counts only: atomics are order-free here), then its tiles stably
// sorted by local pixel (one stable_rank pass for S <= 9 bits, else two LSD
// digit passes) and written out in pixel order; the next tile's events are
// loaded while the current one is sorted.  Every pixel's events keep their
// stream order: the bucketing is a stable sort by pixel (deterministic).
__global__ void __launch_bounds__(1024) bucket_fine_kernel(const uint32_t* __restrict__ temp, const uint32_t* table,
                                                          long long npix, int S, long long nch, int NB,
                                                          uint32_t* offsets, uint16_t* out) {
  extern __shared__ uint32_t bk_smem[];
  const int P = 1 << S;
  const int d1 = S <= 9 ? S : S - S / 2;  // LSD digits: low d1 bits, then S - d1
  const int d2 = S - d1;
  uint32_t* cur = bk_smem;             // [P] global cursor of each local pixel
  uint32_t* tc = cur + P;              // [P] tile counts
  uint32_t* toff = tc + P;             // [P] first tile position of each local pixel
  uint32_t* sbuf = toff + P;           // [BK_TILE] the tile sorted by local pixel
  uint32_t* sbuf2 = sbuf + BK_TILE;    // [BK_TILE] after the first LSD digit (S > 9)
  uint32_t* cnt = sbuf2 + BK_TILE;     // [2^max(d1, d2) * 33] stable-rank counters
  uint32_t* pm = cnt + (33 << (d1 > d2 ? d1 : d2));  // [32][2^max(d1, d2)] peer masks
  __shared__ uint32_t wsum[32];
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bs = table[(long long)b * nch], be = table[(long long)(b + 1) * nch];
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    cur[i] = 0u;
    tc[i] = 0u;
  }
  __syncthreads();
  for (uint32_t i0 = bs + threadIdx.x; i0 < be; i0 += 8 * blockDim.x) {  // 8 loads in flight per thread
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint32_t i = i0 + q * blockDim.x;
      w[q] = i < be ? __ldcg(temp + i) : 0xffffffffu;
    }
#pragma unroll
    for (int q = 0; q < 8; q++)
      if (w[q] != 0xffffffffu) atomicAdd(&cur[w[q] >> 16], 1u);
  }
  // first tile's loads in flight across the scan
  uint32_t nv[BK_ROWS];
#pragma unroll
  for (int q = 0; q < BK_ROWS; q++) {
    const uint32_t i = bs + 256 * warp + 32 * q + lane;
    nv[q] = i < be ? __ldcs(temp + i) : 0u;
  }
  __syncthreads();
  block_scan_smem(cur, cur, P, wsum);
  const long long p0 = (long long)b << S;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    cur[i] += bs;
    if (p0 + i < npix) offsets[p0 + i] = cur[i];
  }
  if (b == NB - 1 && threadIdx.x == 0) offsets[npix] = be;
  __syncthreads();
  for (uint32_t t0 = bs; t0 < be; t0 += BK_TILE) {
    const int nt = (int)min((uint32_t)BK_TILE, be - t0);
    uint32_t v[BK_ROWS], key[BK_ROWS], pos[BK_ROWS];
    uint32_t vm = 0;
#pragma unroll
    for (int q = 0; q < BK_ROWS; q++) {
      v[q] = nv[q];
      vm |= (uint32_t)(256 * warp + 32 * q + lane < nt) << q;
    }
#pragma unroll
    for (int q = 0; q < BK_ROWS; q++) {
      const uint32_t i = t0 + BK_TILE + 256 * warp + 32 * q + lane;
      nv[q] = i < be ? __ldcs(temp + i) : 0u;
    }
    // tile counts per local pixel (order-free atomics) for the output cursors
#pragma unroll
    for (int q = 0; q < BK_ROWS; q++)
      if ((vm >> q) & 1u) atomicAdd(&tc[v[q] >> 16], 1u);
    // stable sort of the tile by local pixel: LSD over one or two digits
#pragma unroll
    for (int q = 0; q < BK_ROWS; q++) key[q] = (v[q] >> 16) & ((1u << d1) - 1u);
    stable_rank(key, vm, pos, cnt, pm, 1 << d1, wsum);
    uint32_t* first = d2 ? sbuf2 : sbuf;
#pragma unroll
    for (int q = 0; q < BK_ROWS; q++)
      if ((vm >> q) & 1u) first[pos[q]] = v[q];
    __syncthreads();
    if (d2) {  // reload in the first digit's order, rank by the high digit
#pragma unroll
      for (int q = 0; q < BK_ROWS; q++) {
        v[q] = (vm >> q) & 1u ? sbuf2[256 * warp + 32 * q + lane] : 0u;
        key[q] = (v[q] >> (16 + d1)) & ((1u << d2) - 1u);
      }
      stable_rank(key, vm, pos, cnt, pm, 1 << d2, wsum);
#pragma unroll
      for (int q = 0; q < BK_ROWS; q++)
        if ((vm >> q) & 1u) sbuf[pos[q]] = v[q];
    }
    block_scan_smem(tc, toff, P, wsum);  // (syncs) toff[lp]: first position of lp in the sorted tile
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
      const uint32_t w = sbuf[i];
      const uint32_t lp = w >> 16;
      out[cur[lp] + (uint32_t)i - toff[lp]] = (uint16_t)(w & 0xffffu);  // consecutive i, same pixel: consecutive
    }
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      cur[i] += tc[i];
      tc[i] = 0u;
    }
    __syncthreads();
  }
}

// pass C shared memory: cur, tc, toff [2^S] + two sorted tiles + stable-rank counters
static size_t bucket_fine_smem(int S) {
  const int d1 = S <= 9 ? S : S - S / 2, d2 = S - d1;
  const int dmax = d1 > d2 ? d1 : d2;
  return sizeof(uint32_t) * ((size_t)3 * (1u << S) + 2 * (size_t)BK_TILE + ((size_t)65 << dmax));
}

static cudaError_t launch_bucket_two_level(const uint32_t* pix, const uint16_t* bins, unsigned long long nev,
                                          long long npix, uint32_t* offsets, uint16_t* bins_out, uint32_t* scratch,
                                          uint32_t* dropped_out, cudaStream_t s, int num_sms) {
  const int S = bucket_shift(npix);
  const int NB = (int)((npix + (1ll << S) - 1) >> S);
  const long long nch = ((long long)nev + BK_CHUNK - 1) / BK_CHUNK;
  const long long nchv = nch > 0 ? nch : 1;
  const long long tn = (long long)NB * nchv;
  uint32_t* temp = scratch;
  uint32_t* table = temp + nev;             // [tn + 1]
  uint32_t* bsum = table + tn + 1;          // [ceil((tn+1) / SCAN_TILE)]
  const long long nbs = (tn + 1 + SCAN_TILE - 1) / SCAN_TILE;
  uint32_t* misc = bsum + nbs;              // [0] dropped, [1] total
  cudaError_t e = cudaMemsetAsync(table, 0, sizeof(uint32_t) * (size_t)(tn + 1 + nbs + 2), s);
  if (e != cudaSuccess) return e;
  if (nch > 0) coarse_count_kernel<<<(unsigned)nch, 512, 0, s>>>(pix, nev, npix, S, NB, nch, table, misc);
  scan_tiles_kernel<<<(unsigned)((tn + SCAN_TILE - 1) / SCAN_TILE), SCAN_THREADS, 0, s>>>(table, tn, table, bsum);
  scan_bsum_kernel<<<1, SCAN_THREADS, 0, s>>>(bsum, (tn + SCAN_TILE - 1) / SCAN_TILE, misc + 1);
  long long fg = (tn + 1 + 255) / 256;
  if (fg > (long long)num_sms * 16) fg = (long long)num_sms * 16;
  scan_add_kernel<<<(unsigned)fg, 256, 0, s>>>(table, bsum, tn, misc + 1);
  const size_t psmem = sizeof(uint32_t) * ((size_t)BK_MAX_BUCKETS * 65 + BK_TILE) + sizeof(uint16_t) * BK_TILE;
  static SmemAttrOnce attr_p, attr_f;  // both at their maximum sizes
  e = smem_attr_once(attr_p, partition_kernel, (int)psmem);
  if (e != cudaSuccess) return e;
  size_t fmax = 0;  // bucket_fine_smem(S) is not monotonic in S
  for (int S2 = 0; S2 <= BK_MAX_S; S2++) fmax = bucket_fine_smem(S2) > fmax ? bucket_fine_smem(S2) : fmax;
  e = smem_attr_once(attr_f, bucket_fine_kernel, (int)fmax);
  if (e != cudaSuccess) return e;
  if (nch > 0) partition_kernel<<<(unsigned)nch, 1024, psmem, s>>>(pix, bins, nev, npix, S, NB, nch, table, temp);
  // with no events the table is all zeros: pass C writes zero offsets
  const size_t smem = bucket_fine_smem(S);
  bucket_fine_kernel<<<(unsigned)NB, 1024, smem, s>>>(temp, table, npix, S, nchv, NB, offsets, bins_out);
  if (dropped_out) {
    e = cudaMemcpyAsync(dropped_out, misc, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

static cudaError_t launch_bucket_atomic(const uint32_t* pix, const uint16_t* bins, unsigned long long nev,
                                        long long npix, uint32_t* offsets, uint16_t* bins_out, uint32_t* scratch,
                                        uint32_t* dropped_out, cudaStream_t s, int num_sms) {
  const long long nb = (npix + SCAN_TILE - 1) / SCAN_TILE;
  uint32_t* cnt = scratch;            // [npix]: counts, then cursors
  uint32_t* bsum = scratch + npix;    // [nb]
  uint32_t* misc = bsum + nb;         // [0] dropped, [1] total
  cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * ((size_t)npix + (size_t)nb + 2), s);
  if (e != cudaSuccess) return e;
  const long long ev_grid = (long long)num_sms * 8;
  if (nev) count_kernel<<<(unsigned)ev_grid, 256, 0, s>>>(pix, nev, npix, cnt, misc);
  if (npix > 0) {
    scan_tiles_kernel<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(cnt, npix, offsets, bsum);
    scan_bsum_kernel<<<1, SCAN_THREADS, 0, s>>>(bsum, nb, misc + 1);
  }
  long long fg = (npix + 1 + 255) / 256;
  if (fg > (long long)num_sms * 16) fg = (long long)num_sms * 16;
  scan_fix_kernel<<<(unsigned)fg, 256, 0, s>>>(offsets, cnt, bsum, npix, misc + 1);
  if (nev) scatter_kernel<<<(unsigned)ev_grid, 256, 0, s>>>(pix, bins, nev, npix, cnt, bins_out);
  if (dropped_out) {
    e = cudaMemcpyAsync(dropped_out, misc, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_bucket(const uint32_t* pix, const uint16_t* bins, unsigned long long nev, long long npix,
                          uint32_t* offsets, uint16_t* bins_out, uint32_t* scratch, uint32_t* dropped_out,
                          cudaStream_t s, int num_sms) {
  if (bucket_two_level(npix))
    return launch_bucket_two_level(pix, bins, nev, npix, offsets, bins_out, scratch, dropped_out, s, num_sms);
  return launch_bucket_atomic(pix, bins, nev, npix, offsets, bins_out, scratch, dropped_out, s, num_sms);
}

}  // namespace srt3d
