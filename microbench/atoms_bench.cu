// Shared-memory atomic throughput on sm_100a (for the bin-count sketch path):
// atomicAdd(&hist[x], 1) on a 4096-bin uint32 histogram, x uniform random or
// half of them in a 24-bin cluster (Gaussian-ish surface), 512-thread CTAs,
// 2 CTAs / SM.  Reports atomics per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ unsigned long long g_cyc[4096];
template <int MODE>
__global__ void __launch_bounds__(512) k(unsigned* out, int iters) {
  extern __shared__ unsigned hist[];
  for (int i = threadIdx.x; i < 4096 * 4; i += blockDim.x) hist[i] = 0;
  const unsigned rep = (MODE == 3) ? ((threadIdx.x & 1) << 12) : (MODE == 4) ? ((threadIdx.x & 3) << 12) :
                       (MODE == 5) ? (((threadIdx.x >> 5) & 3) << 12) : 0u;
  __syncthreads();
  unsigned s = threadIdx.x * 2654435761u + blockIdx.x * 40503u + 1;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      s = s * 1664525u + 1013904223u;
      unsigned x = s >> 20;                       // uniform 0..4095
      if (MODE != 0 && MODE != 2 && (s & 0x80000u)) x = 2000u + ((s >> 8) & 15u) + ((s >> 12) & 7u);  // 50% in ~24 bins
      if (MODE == 2) { hist[x] += 1u; } else atomicAdd(&hist[x + rep], 1u);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  unsigned acc = 0;
  for (int i = threadIdx.x; i < 4096 * 4; i += blockDim.x) acc += hist[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char* name, int nsm, unsigned* out) {
  const int iters = 2000, blocks = nsm * 2;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<MODE><<<blocks, 512, 65536>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 512, 65536>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double total = (double)blocks * 512 * iters * 8;
  printf("{\"test\":\"%s\",\"atomics_per_s\":%.3e,\"per_clk_per_sm_at_1.92GHz\":%.2f,\"ms\":%.3f}\n", name, total / (ms * 1e-3),
         total / (ms * 1e-3) / nsm / 1.92e9, ms);
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out; cudaMalloc(&out, sizeof(unsigned) * nsm * 2 * 512);
  run<0>("atoms_uniform", nsm, out);
  run<1>("atoms_half_clustered", nsm, out);
  run<2>("lds_sts_nonatomic_uniform", nsm, out);
  run<3>("atoms_clustered_2copies_by_lane", nsm, out);
  run<4>("atoms_clustered_4copies_by_lane", nsm, out);
  run<5>("atoms_clustered_4copies_by_warp", nsm, out);
  return 0;
}
