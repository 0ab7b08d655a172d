// tcgen05.mma issue-to-completion rate on sm_100a for the operand configurations the
// tensor-core sketch uses: kind::f16, M = 128, N = 128, K = 16 per instruction,
// one CTA per SM, one thread issuing `iters` MMAs into one TMEM accumulator, then one commit;
// cycles per MMA from clock64 around issue + mbarrier wait.  Operands are zeros (the rate does
// not depend on values).  Variants:
//   ss_ns   : A and B in shared memory, SWIZZLE_NONE K-major (LBO 128 B, SBO 16 Kb)
//   ss_sw   : A and B in shared memory, SWIZZLE_128B K-major
//   ts_ns   : A in TMEM, B in shared memory SWIZZLE_NONE
//   ts_sw   : A in TMEM, B SWIZZLE_128B
// With `lsu`=1 the other warps of the CTA stream 16-byte shared stores (zeroing traffic) meanwhile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench/umma_rate microbench/umma_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                     \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, bool sw, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(sw ? 1 : (128 >> 4)) << 16;
  d |= (uint64_t)(((sw ? 1024u : sbo) >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  if (sw) d |= (uint64_t)2 << 61;
  return d;
}

__device__ unsigned long long g_cyc[1024];

__global__ void __launch_bounds__(256, 1) k_umma(int variant, int iters, int lsu, int N, int M) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const bool ts = variant >= 2, sw = variant & 1;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 2 * 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const uint32_t Kb = 256, sbo = 16 * Kb;
  const uint32_t sa = su32(sm), sb = su32(sm + 65536);
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      const uint32_t kk = it & 15;
      const uint32_t off = sw ? (kk >> 2) * 16384 + (kk & 3) * 32 : kk * 256;
      const uint64_t bd = desc(sb + off, sw, sbo);
      if (ts) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
            "r"(tmem + 256 + kk * 8), "l"(bd), "r"(idesc), "r"(it > 0 ? 1 : 0));
      } else {
        const uint64_t ad = desc(sa + off, sw, sbo);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(it > 0 ? 1 : 0));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
            su32(&bar))
        : "memory");
    g_cyc[blockIdx.x] = (unsigned long long)(clock64() - t0);
    done = 1;
  } else if (lsu && warp >= 1) {
    // zeroing traffic into a third 64 KB region while the MMAs run
    uint4* z = reinterpret_cast<uint4*>(sm + 131072);
    while (!done)
      for (int i = tid - 32; i < 65536 / 16; i += blockDim.x - 32) z[i] = make_uint4(0, 0, 0, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = 1024 + 3 * 65536;
  CK(cudaFuncSetAttribute(k_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const char* names[4] = {"ss_ns", "ss_sw", "ts_ns", "ts_sw"};
  const int iters = 4096;
  const int shapes[5][2] = {{128, 128}, {256, 128}, {64, 128}, {128, 64}, {256, 64}};
  for (int sh = 0; sh < 5; sh++)
  for (int lsu = 0; lsu < (sh == 0 ? 2 : 1); lsu++)
    for (int v = 0; v < 4; v++) {
      const int N = shapes[sh][0], M = shapes[sh][1];
      k_umma<<<nsm, 256, smem>>>(v, iters, lsu, N, M);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      unsigned long long c[1024];
      CK(cudaMemcpyFromSymbol(c, g_cyc, sizeof(unsigned long long) * nsm));
      double s = 0;
      for (int i = 0; i < nsm; i++) s += (double)c[i];
      printf("{\"variant\": \"%s\", \"M\": %d, \"N\": %d, \"lsu_traffic\": %d, \"cycles_per_mma\": %.1f, "
             "\"flops_per_clk\": %.0f}\n", names[v], M, N, lsu, s / nsm / iters, 2.0 * M * N * 16 / (s / nsm / iters));
    }
  return 0;
}
