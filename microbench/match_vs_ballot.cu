// Warp peer-mask of 9-bit keys: __match_any_sync vs 9 ballots (timing only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ uint32_t g_sink;
__global__ void k_match(int iters) {
  uint32_t key = (threadIdx.x * 2654435761u) >> 23, acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const uint32_t k = (key + r * 77u) & 511u;
      acc += __popc(__match_any_sync(0xffffffffu, k) & ((1u << (threadIdx.x & 31)) - 1u));
    }
    key = key * 1664525u + 1013904223u;
  }
  if (acc == 0xdeadbeef) g_sink = acc;
}
__global__ void k_ballot(int iters) {
  uint32_t key = (threadIdx.x * 2654435761u) >> 23, acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const uint32_t k = (key + r * 77u) & 511u;
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 9; b++) {
        const bool bit = (k >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
      acc += __popc(peers & ((1u << (threadIdx.x & 31)) - 1u));
    }
    key = key * 1664525u + 1013904223u;
  }
  if (acc == 0xdeadbeef) g_sink = acc;
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int t = 0; t < 2; t++) {
    const int iters = 2000;
    if (t == 0) k_match<<<nsm * 2, 1024>>>(10); else k_ballot<<<nsm * 2, 1024>>>(10);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    if (t == 0) k_match<<<nsm * 2, 1024>>>(iters); else k_ballot<<<nsm * 2, 1024>>>(iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ev = (double)nsm * 2 * 1024 * iters * 8;
    printf("%s: %.3f ms, %.3e keys/s, %.2f warp-rows/clk/SM\n", t == 0 ? "match_any" : "ballot9", ms, ev / (ms * 1e-3),
           ev / 32 / (ms * 1e-3) / nsm / 1.965e9);
  }
  return 0;
}
