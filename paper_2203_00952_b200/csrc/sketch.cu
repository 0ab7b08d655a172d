// K1 dispatch + debug/validation kernels (see sketch_impl.cuh for K1 itself).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace srt3d {

cudaError_t launch_sketch_g4(int M, bool tab, const SketchArgs& a, cudaStream_t s, int num_sms);
cudaError_t launch_sketch_g8(int M, bool tab, const SketchArgs& a, cudaStream_t s, int num_sms);
cudaError_t launch_sketch_g16(int M, bool tab, const SketchArgs& a, cudaStream_t s, int num_sms);
cudaError_t launch_sketch_g32(int M, bool tab, const SketchArgs& a, cudaStream_t s, int num_sms);
cudaError_t launch_sketch_g4_cheb(int M, const SketchArgs& a, cudaStream_t s, int num_sms);

// ---- debug / validation kernels -----------------------------------------
__global__ void phase_index_kernel(const uint16_t* __restrict__ bins, long long n, uint32_t T, uint32_t m,
                                   uint32_t* __restrict__ r) {
  const float invT = 1.0f / (float)T;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const uint32_t x = bins[p];
    for (uint32_t j = 1; j <= m; j++) r[(size_t)p * m + (j - 1)] = phase_index(x, j, T, invT);
  }
}

__global__ void check_csr_kernel(const uint16_t* __restrict__ bins, const uint32_t* __restrict__ offsets,
                                 long long npix, uint32_t T, int32_t* bad) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += stride) {
    const uint32_t b = offsets[i], e = offsets[i + 1];
    if (e < b) {
      atomicOr(bad, 1);
      continue;
    }
    for (uint32_t p = b; p < e; p++)
      if (bins[p] >= T) {
        atomicOr(bad, 2);
        break;
      }
  }
}

// K8: the FP32 FMA rate this GPU sustains right now — 8
// independent FFMA chains per thread, 1024-thread CTAs, 4 per SM; the
// roofline's "also measure it in the same run".
__global__ void __launch_bounds__(1024) ffma_peak_kernel(float* out, float b, float c, int iters) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; i++) v[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < 8; i++) v[i] = fmaf(v[i], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; i++) s += v[i];
  if (s == 12345.678f) out[0] = s;  // keeps the chains live
}

cudaError_t measure_ffma_peak(double* tflops, int num_sms) {
  float* dummy = nullptr;
  cudaEvent_t e0, e1;
  cudaError_t e = cudaMalloc(&dummy, sizeof(float));
  if (e != cudaSuccess) return e;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, blocks = num_sms * 2, threads = 1024;
  ffma_peak_kernel<<<blocks, threads>>>(dummy, 0.999f, 1e-3f, 64);  // warm-up
  cudaEventRecord(e0);
  ffma_peak_kernel<<<blocks, threads>>>(dummy, 0.999f, 1e-3f, iters);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  if (e == cudaSuccess) *tflops = 2.0 * 8 * 16 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(dummy);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t launch_sketch_pass(int M, int G, const SketchArgs& a, cudaStream_t s, int num_sms) {
  const bool tab = ((size_t)a.T + 1) * sizeof(float2) <= SK_MAX_SMEM;
  if (!tab) return launch_sketch_g32(M, false, a, s, num_sms);
  if (G == SK_G4_CHEB) return launch_sketch_g4_cheb(M, a, s, num_sms);
  switch (G) {
    case 4:
      return launch_sketch_g4(M, true, a, s, num_sms);
    case 8:
      return launch_sketch_g8(M, true, a, s, num_sms);
    case 16:
      return launch_sketch_g16(M, true, a, s, num_sms);
    default:
      return launch_sketch_g32(M, true, a, s, num_sms);
  }
}

cudaError_t launch_phase_index(const uint16_t* bins, long long n, uint32_t T, uint32_t m, uint32_t* r,
                               cudaStream_t s, int num_sms) {
  long long grid = (n + 255) / 256;
  if (grid > (long long)num_sms * 8) grid = (long long)num_sms * 8;
  if (grid < 1) grid = 1;
  phase_index_kernel<<<(unsigned)grid, 256, 0, s>>>(bins, n, T, m, r);
  return cudaGetLastError();
}

cudaError_t launch_check_csr(const uint16_t* bins, const uint32_t* offsets, long long npix, uint32_t T,
                             int32_t* bad, cudaStream_t s, int num_sms) {
  long long grid = (npix + 255) / 256;
  if (grid > (long long)num_sms * 8) grid = (long long)num_sms * 8;
  if (grid < 1) grid = 1;
  check_csr_kernel<<<(unsigned)grid, 256, 0, s>>>(bins, offsets, npix, T, bad);
  return cudaGetLastError();
}

}  // namespace srt3d
