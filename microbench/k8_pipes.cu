// K8 roofline microbenchmarks for sm_100a:
// measure FP32-pipe lane-op rates for scalar FFMA/FADD/FMUL and packed
// FFMA2/FADD2/FMUL2, the MUFU (XU) sin/cos rate, random-index LDS.64 rate,
// the two candidate sketch inner loops (complex-power recurrence and the
// packed Chebyshev recurrence), and HBM copy bandwidth.
// Each test launches one 1024-thread CTA per SM, reads clock64() around the
// body and reports lane-ops per clock per SM plus the effective SM clock.
#include <cstdio>
#include <string>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float2 upk(u64 v) { float2 r; asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) { u64 d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }

__device__ unsigned long long g_cycles[4096];

#define NCH 8
// scalar FFMA: 8 independent chains, 3-register form
__global__ void k_ffma(float* out, float b, float c, int iters) {
  float a[NCH]; for (int i = 0; i < NCH; i++) a[i] = threadIdx.x * 1e-3f + i;
  float bb = b + threadIdx.x * 1e-9f, cc = c - threadIdx.x * 1e-9f;
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < NCH; i++) a[i] = fmaf(a[i], bb, cc);
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; i++) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
__global__ void k_fadd(float* out, float b, float c, int iters) {
  float a[NCH]; for (int i = 0; i < NCH; i++) a[i] = threadIdx.x * 1e-3f + i;
  float bb = b + threadIdx.x * 1e-9f;
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < NCH; i++) a[i] = a[i] + bb;
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; i++) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// packed FFMA2: 8 independent packed chains
__global__ void k_ffma2(float* out, float b, float c, int iters) {
  u64 a[NCH]; for (int i = 0; i < NCH; i++) a[i] = pk(threadIdx.x * 1e-3f + i, i * 0.5f);
  u64 bb = pk(b + threadIdx.x * 1e-9f, b), cc = pk(c, c - threadIdx.x * 1e-9f);
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < NCH; i++) a[i] = ffma2(a[i], bb, cc);
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; i++) { float2 v = upk(a[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
__global__ void k_fadd2(float* out, float b, float c, int iters) {
  u64 a[NCH]; for (int i = 0; i < NCH; i++) a[i] = pk(threadIdx.x * 1e-3f + i, i * 0.5f);
  u64 bb = pk(b + threadIdx.x * 1e-9f, b);
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < NCH; i++) a[i] = fadd2(a[i], bb);
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; i++) { float2 v = upk(a[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// MUFU sin+cos (XU pipe): __sinf/__cosf on independent values
__global__ void k_mufu(float* out, float b, float c, int iters) {
  float a[NCH]; for (int i = 0; i < NCH; i++) a[i] = threadIdx.x * 1e-3f + i;
  float acc = 0;
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NCH; i++) { float s, co; asm volatile("sin.approx.f32 %0, %1;" : "=f"(s) : "f"(a[i])); asm volatile("cos.approx.f32 %0, %1;" : "=f"(co) : "f"(a[i])); a[i] = s + co; }
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; i++) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// sketch inner loop, packed complex-power recurrence: per term FMUL2+FFMA2 (p*=w) + FADD2 (S+=p)
template <int M>
__global__ void k_cplx2(float* out, float b, float c, int iters) {
  u64 S[M]; for (int j = 0; j < M; j++) S[j] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  u64 W = pk(wr, wi), Wn = pk(-wi, wr);
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
    u64 p = W;
#pragma unroll
    for (int j = 0; j < M; j++) {
      S[j] = fadd2(S[j], p);
      float2 pv = upk(p);
      p = ffma2(pk(pv.y, pv.y), Wn, fmul2(pk(pv.x, pv.x), W));
    }
    W = fadd2(W, pk(1e-7f, -1e-7f)); Wn = pk(-upk(W).y, upk(W).x);
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int j = 0; j < M; j++) { float2 v = upk(S[j]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// sketch inner loop, scalar complex recurrence: 2 FMUL + 2 FFMA + 2 FADD per term
template <int M>
__global__ void k_cplx1(float* out, float b, float c, int iters) {
  float Sr[M], Si[M]; for (int j = 0; j < M; j++) { Sr[j] = 0; Si[j] = 0; }
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
    float pr = wr, pi = wi;
#pragma unroll
    for (int j = 0; j < M; j++) {
      Sr[j] += pr; Si[j] += pi;
      float nr = fmaf(pr, wr, -pi * wi); float ni = fmaf(pr, wi, pi * wr);
      pr = nr; pi = ni;
    }
    wr += 1e-7f; wi -= 1e-7f;
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int j = 0; j < M; j++) s += Sr[j] + Si[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// sketch inner loop, packed Chebyshev: Y_{j+1} = (-2c) Y_j + Y_{j-1} (sign-alternating form), S_j += Y_j
template <int M>
__global__ void k_cheb2(float* out, float b, float c, int iters) {
  u64 S[M]; for (int j = 0; j < M; j++) S[j] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
    u64 y0 = pk(1.f, 0.f), y1 = pk(-wr, -wi);
    float n2c = -2.f * wr;
    u64 C = pk(n2c, n2c);
#pragma unroll
    for (int j = 0; j < M; j++) {
      S[j] = fadd2(S[j], y1);
      u64 y2 = ffma2(C, y1, y0); y0 = y1; y1 = y2;
    }
    wr += 1e-7f; wi -= 1e-7f;
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int j = 0; j < M; j++) { float2 v = upk(S[j]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// random-index LDS.64 from an 8192-entry float2 table
__global__ void k_lds(float* out, float b, float c, int iters) {
  __shared__ float2 tab[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = make_float2(i, -i);
  __syncthreads();
  unsigned r[NCH]; for (int i = 0; i < NCH; i++) r[i] = (threadIdx.x * 2654435761u + i * 40503u) & 4095u;
  float2 acc = make_float2(0, 0);
  u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NCH; i++) { float2 v = tab[r[i]]; acc.x += v.x; acc.y += v.y; r[i] = (r[i] + 2897u + (unsigned)it) & 4095u; }
  }
  __syncthreads(); u64 t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// mixed: 8 packed FFMA2 chains + 8 scalar FFMA chains per thread (can heavy+lite run concurrently?)
__global__ void k_mix_ffma2_ffma(float* out, float b, float c, int iters) {
  u64 a[NCH]; float s[NCH];
  for (int i = 0; i < NCH; i++) { a[i] = pk(threadIdx.x * 1e-3f + i, i * 0.5f); s[i] = threadIdx.x * 1e-3f - i; }
  u64 bb = pk(b + threadIdx.x * 1e-9f, b), cc = pk(c, c - threadIdx.x * 1e-9f);
  float sb = b - threadIdx.x * 1e-9f, sc = c + threadIdx.x * 1e-9f;
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < NCH; i++) { a[i] = ffma2(a[i], bb, cc); s[i] = fmaf(s[i], sb, sc); }
  }
  __syncthreads(); u64 t1 = clock64();
  float r = 0; for (int i = 0; i < NCH; i++) { float2 v = upk(a[i]); r += v.x + v.y + s[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// mixed: 2 packed FFMA2 per 1 scalar FFMA
__global__ void k_mix_2ffma2_1ffma(float* out, float b, float c, int iters) {
  u64 a[NCH]; float s[NCH];
  for (int i = 0; i < NCH; i++) { a[i] = pk(threadIdx.x * 1e-3f + i, i * 0.5f); s[i] = threadIdx.x * 1e-3f - i; }
  u64 bb = pk(b + threadIdx.x * 1e-9f, b), cc = pk(c, c - threadIdx.x * 1e-9f);
  float sb = b - threadIdx.x * 1e-9f, sc = c + threadIdx.x * 1e-9f;
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < NCH; i++) { a[i] = ffma2(a[i], bb, cc); if (i & 1) s[i] = fmaf(s[i], sb, sc); }
  }
  __syncthreads(); u64 t1 = clock64();
  float r = 0; for (int i = 0; i < NCH; i++) { float2 v = upk(a[i]); r += v.x + v.y + s[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// mixed FADD2 + scalar FFMA
__global__ void k_mix_fadd2_ffma(float* out, float b, float c, int iters) {
  u64 a[NCH]; float s[NCH];
  for (int i = 0; i < NCH; i++) { a[i] = pk(threadIdx.x * 1e-3f + i, i * 0.5f); s[i] = threadIdx.x * 1e-3f - i; }
  u64 bb = pk(b + threadIdx.x * 1e-9f, b);
  float sb = b - threadIdx.x * 1e-9f, sc = c + threadIdx.x * 1e-9f;
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int i = 0; i < NCH; i++) { a[i] = fadd2(a[i], bb); s[i] = fmaf(s[i], sb, sc); }
  }
  __syncthreads(); u64 t1 = clock64();
  float r = 0; for (int i = 0; i < NCH; i++) { float2 v = upk(a[i]); r += v.x + v.y + s[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// scalar complex recurrence with scalar accumulate, 2 photon chains (ILP2), sketch-like
template <int M>
__global__ void k_cplx1x2(float* out, float b, float c, int iters) {
  float Sr[M], Si[M]; for (int j = 0; j < M; j++) { Sr[j] = 0; Si[j] = 0; }
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  float vr = cosf(threadIdx.x * 2e-3f), vi = sinf(threadIdx.x * 2e-3f);
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
    float pr = wr, pi = wi, qr = vr, qi = vi;
#pragma unroll
    for (int j = 0; j < M; j++) {
      Sr[j] += pr + qr; Si[j] += pi + qi;
      float nr = fmaf(pr, wr, -pi * wi); float ni = fmaf(pr, wi, pi * wr);
      float mr = fmaf(qr, vr, -qi * vi); float mi = fmaf(qr, vi, qi * vr);
      pr = nr; pi = ni; qr = mr; qi = mi;
    }
    wr += 1e-7f; wi -= 1e-7f; vr -= 1e-7f; vi += 1e-7f;
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int j = 0; j < M; j++) s += Sr[j] + Si[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
// packed recurrence (FMUL2+FFMA2) but scalar accumulation FADD (lite pipe?), 2 chains
template <int M>
__global__ void k_cplx2_acc1(float* out, float b, float c, int iters) {
  float Sr[M], Si[M]; for (int j = 0; j < M; j++) { Sr[j] = 0; Si[j] = 0; }
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  float vr = cosf(threadIdx.x * 2e-3f), vi = sinf(threadIdx.x * 2e-3f);
  u64 W = pk(wr, wi), Wn = pk(-wi, wr), V = pk(vr, vi), Vn = pk(-vi, vr);
  __syncthreads(); u64 t0 = clock64();
  for (int it = 0; it < iters; it++) {
    u64 p = W, q = V;
#pragma unroll
    for (int j = 0; j < M; j++) {
      float2 pv = upk(p), qv = upk(q);
      Sr[j] += pv.x; Si[j] += pv.y; Sr[j] += qv.x; Si[j] += qv.y;
      p = ffma2(pk(pv.y, pv.y), Wn, fmul2(pk(pv.x, pv.x), W));
      q = ffma2(pk(qv.y, qv.y), Vn, fmul2(pk(qv.x, qv.x), V));
    }
    W = fadd2(W, pk(1e-7f, -1e-7f)); Wn = pk(-upk(W).y, upk(W).x);
    V = fadd2(V, pk(-1e-7f, 1e-7f)); Vn = pk(-upk(V).y, upk(V).x);
  }
  __syncthreads(); u64 t1 = clock64();
  float s = 0; for (int j = 0; j < M; j++) s += Sr[j] + Si[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}
__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

typedef void (*kfn)(float*, float, float, int);
static void run(const char* name, kfn f, int iters, double lane_ops_per_iter_per_thread, int nsm, float* out, int bs = 1024) {
  dim3 grid(nsm * (1024 / bs)), block(bs);
  f<<<grid, block>>>(out, 1.0000001f, 1e-7f, 8);  // warm
  CK(cudaGetLastError());  // launch failures (e.g. resources) must not read as a 0-ms run
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  f<<<grid, block>>>(out, 1.0000001f, 1e-7f, iters);
  CK(cudaGetLastError());
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long cyc[4096];
  int nb = nsm * (1024 / bs);
  CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(u64) * nb));
  double mx = 0, mean = 0; for (int i = 0; i < nb; i++) { mean += cyc[i]; if (cyc[i] > mx) mx = cyc[i]; }
  mean /= nb;
  // rates from the event-timed total (valid whatever the residency); per clock at the 1965 MHz max
  // clock the pool runs these at (no throttle reasons), and the clock64 view when all blocks of an
  // SM are co-resident (1024 threads per SM)
  double total = lane_ops_per_iter_per_thread * iters * (double)bs * (double)nb / (ms * 1e-3);
  double per_clk = total / (nsm * 1.965e9);
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, bs, 0));
  const bool resident = per_sm * bs >= 1024;
  printf("{\"test\":\"%s\",\"lane_ops_per_clk_per_sm\":%.2f,\"lane_ops_per_s\":%.4e,\"ms\":%.3f,"
         "\"resident_blocks_per_sm\":%d,\"clock64_eff_ghz\":%s}\n", name, per_clk, total, ms, per_sm,
         resident ? std::to_string(mx / (ms * 1e6)).c_str() : "null");
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  int l2; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  printf("{\"sms\":%d,\"max_clock_khz\":%d,\"l2_bytes\":%d}\n", nsm, clk, l2);
  float* out; CK(cudaMalloc(&out, sizeof(float) * nsm * 1024));
  const int IT = 4000;
  run("ffma_scalar", k_ffma, IT, 16.0 * NCH, nsm, out);       // 1 lane-op (FFMA) per instruction
  run("fadd_scalar", k_fadd, IT, 16.0 * NCH, nsm, out);
  run("ffma2_packed", k_ffma2, IT, 16.0 * NCH * 2, nsm, out);   // 2 lane-ops per FFMA2
  run("fadd2_packed", k_fadd2, IT, 16.0 * NCH * 2, nsm, out);
  run("mufu_sin_cos", k_mufu, IT, NCH * 2.0, nsm, out);         // MUFU ops
  // sketch loops: report TERMS (photon x frequency) per clk per SM
  run("sketch_cplx2_m32_terms", k_cplx2<32>, IT / 4, 32.0, nsm, out, 256);
  run("sketch_cplx1_m32_terms", k_cplx1<32>, IT / 4, 32.0, nsm, out, 256);
  run("sketch_cheb2_m32_terms", k_cheb2<32>, IT / 4, 32.0, nsm, out, 256);
  run("sketch_cplx1x2_m32_terms", k_cplx1x2<32>, IT / 4, 64.0, nsm, out, 256);
  run("sketch_cplx2acc1_m32_terms", k_cplx2_acc1<32>, IT / 4, 64.0, nsm, out, 256);
  run("sketch_cplx1x2_m16_terms", k_cplx1x2<16>, IT / 2, 32.0, nsm, out, 512);
  run("sketch_cplx2acc1_m16_terms", k_cplx2_acc1<16>, IT / 2, 32.0, nsm, out, 512);
  run("mix_ffma2_ffma", k_mix_ffma2_ffma, IT, 16.0 * NCH * 3, nsm, out);
  run("mix_2ffma2_1ffma", k_mix_2ffma2_1ffma, IT, 16.0 * NCH * 2.5, nsm, out);
  run("mix_fadd2_ffma", k_mix_fadd2_ffma, IT, 16.0 * NCH * 3, nsm, out);
  run("sketch_cplx2_m10_terms", k_cplx2<10>, IT, 10.0, nsm, out);
  run("sketch_cheb2_m10_terms", k_cheb2<10>, IT, 10.0, nsm, out);
  run("lds64_random", k_lds, IT, NCH, nsm, out);
  // HBM copy
  size_t n = (size_t)1 << 27;  // 2 GiB per buffer of uint4
  uint4 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  CK(cudaMemset(a, 1, n * 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 6; r++) {
    cudaEventRecord(e0); k_copy<<<nsm * 8, 512>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r > 0 && ms < best) best = ms;
  }
  printf("{\"test\":\"copy_gbs\",\"gbs\":%.1f}\n", 2.0 * n * 16 / (best * 1e-3) / 1e9);
  return 0;
}
