// NEXT-4 — streaming acquisition: the sketch "can be updated
// in an online fashion with each incoming photon".
//
//   srt3d_sketch_merge: z = (n_a z_a + n_b z_b) / (n_a + n_b), n = n_a + n_b
//      — folds the sketch of a new photon batch into a running
//     sketch; in place (z_out = z_a, n_out = n_a) is allowed.
//   srt3d_bucket_events: an unsorted (pixel, bin) event stream -> the
//     pixel-sorted CSR frame srt3d_sketch consumes (reading A21): count per
//     pixel (global atomics), exclusive scan (block scan + scan of block sums
//     + fix-up), scatter (atomic cursors).  The order of a pixel's bins follows
//     atomic arrival, so the CSR is a valid permutation of the stable sort (the
//     sketch is order-invariant up to fp32 rounding); offsets are exact.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace srt3d {

// One warp per pixel: counts are read before the (possibly aliased) count
// output is written; the row's m complex values are spread over the lanes.
__global__ void __launch_bounds__(256) merge_kernel(const float2* __restrict__ za, const uint32_t* na,
                                                    const float2* __restrict__ zb, const uint32_t* nb,
                                                    long long npix, uint32_t m, float2* zo, uint32_t* no) {
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < npix; i += nw) {
    const uint32_t a = na[i], b = nb[i];
    const uint64_t n = (uint64_t)a + b;
    const double inv = n ? 1.0 / (double)n : 0.0;
    const float wa = (float)((double)a * inv), wb = (float)((double)b * inv);
    for (uint32_t j = lane; j < m; j += 32) {
      const float2 x = za[(size_t)i * m + j], y = zb[(size_t)i * m + j];
      zo[(size_t)i * m + j] = make_float2(fmaf(wa, x.x, wb * y.x), fmaf(wa, x.y, wb * y.y));
    }
    __syncwarp();
    if (lane == 0) no[i] = (uint32_t)n;
  }
}

cudaError_t launch_merge(const float* za, const uint32_t* na, const float* zb, const uint32_t* nb, long long npix,
                         uint32_t m, float* zo, uint32_t* no, cudaStream_t s, int num_sms) {
  if (npix <= 0) return cudaSuccess;
  long long grid = (npix + 7) / 8;
  if (grid > (long long)num_sms * 16) grid = (long long)num_sms * 16;
  merge_kernel<<<(unsigned)grid, 256, 0, s>>>(reinterpret_cast<const float2*>(za), na,
                                              reinterpret_cast<const float2*>(zb), nb, npix, m,
                                              reinterpret_cast<float2*>(zo), no);
  return cudaGetLastError();
}

// ---- bucketing --------------------------------------------------------------
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_PER_THREAD = 4;
constexpr long long SCAN_TILE = (long long)SCAN_THREADS * SCAN_PER_THREAD;

size_t bucket_scratch_words(long long npix) {
  const long long nb = (npix + SCAN_TILE - 1) / SCAN_TILE;
  return (size_t)npix + (size_t)nb + 2;  // counts/cursors, block sums, dropped
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

cudaError_t launch_bucket(const uint32_t* pix, const uint16_t* bins, unsigned long long nev, long long npix,
                          uint32_t* offsets, uint16_t* bins_out, uint32_t* scratch, uint32_t* dropped_out,
                          cudaStream_t s, int num_sms) {
  const long long nb = (npix + SCAN_TILE - 1) / SCAN_TILE;
  uint32_t* cnt = scratch;            // [npix]: counts, then cursors
  uint32_t* bsum = scratch + npix;    // [nb]
  uint32_t* misc = bsum + nb;         // [0] dropped, [1] total
  cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * bucket_scratch_words(npix), s);
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

}  // namespace srt3d
