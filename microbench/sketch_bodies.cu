// Sketch inner-loop bodies on sm_100a (timing only; values are garbage).
// Each thread runs `iters` photons through an M = 32 frequency body and
// accumulates into per-thread sums; we report photon-terms per clock per SM
// (the FP32 roofline of the 8-flop term is 32 terms/clk/SM: 128 FMA lanes,
// 4 lane-ops per Chebyshev term).  Variants:
//   cheb1    : (re, im) pair chain, scalar coefficient, one photon   [shipped body, class-uniform]
//   cheb2p   : same, two photons interleaved (ILP 2)
//   jsplit   : pairs (v_j, v_{j+16}) of one photon: X and Y chains share the
//              scalar coefficient (reuse), S pairs (S_j, S_{j+16})
//   twoslot  : pairs (photon A, photon B) of one component, coefficient pair
//   srpa     : scalar FFMA chains, accumulate (x_j, x_{j+1}) pairs with FADD2
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float2 upk(u64 v) { float2 r; asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 neg2(u64 v) { float2 f = upk(v); return pk(-f.x, -f.y); }

__device__ float g_sink[1];

template <int NT>
__global__ void __launch_bounds__(NT) k_cheb1(float* out, int iters) {
  constexpr int M = 32;
  u64 S[M];
#pragma unroll
  for (int j = 0; j < M; j++) S[j] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  for (int it = 0; it < iters; it++) {
    u64 A = pk(1.f, 0.f), B = pk(wr, wi);
    const u64 C = pk(2.f * wr, 2.f * wr);
#pragma unroll
    for (int j = 0; j < M; j++) {
      if (j) { u64 N = ffma2(B, C, neg2(A)); A = B; B = N; }
      S[j] = fadd2(S[j], B);
    }
    wr += 1e-7f; wi -= 1e-7f;
  }
  float s = 0; for (int j = 0; j < M; j++) { float2 v = upk(S[j]); s += v.x + v.y; }
  if (s == 1234.5f) g_sink[0] = s;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_cheb2p(float* out, int iters) {
  constexpr int M = 32;
  u64 S[M];
#pragma unroll
  for (int j = 0; j < M; j++) S[j] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  float vr = cosf(threadIdx.x * 2e-3f), vi = sinf(threadIdx.x * 2e-3f);
  for (int it = 0; it < iters; it += 2) {
    u64 A = pk(1.f, 0.f), B = pk(wr, wi), A2 = pk(1.f, 0.f), B2 = pk(vr, vi);
    const u64 C = pk(2.f * wr, 2.f * wr), C2 = pk(2.f * vr, 2.f * vr);
#pragma unroll
    for (int j = 0; j < M; j++) {
      if (j) {
        u64 N = ffma2(B, C, neg2(A)); A = B; B = N;
        u64 N2 = ffma2(B2, C2, neg2(A2)); A2 = B2; B2 = N2;
      }
      S[j] = fadd2(S[j], fadd2(B, B2));
    }
    wr += 1e-7f; wi -= 1e-7f; vr -= 1e-7f; vi += 1e-7f;
  }
  float s = 0; for (int j = 0; j < M; j++) { float2 v = upk(S[j]); s += v.x + v.y; }
  if (s == 1234.5f) g_sink[0] = s;
}

// cheb2p with separate accumulation of each photon (2 FADD2 per term pair)
template <int NT>
__global__ void __launch_bounds__(NT) k_cheb2q(float* out, int iters) {
  constexpr int M = 32;
  u64 S[M];
#pragma unroll
  for (int j = 0; j < M; j++) S[j] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  float vr = cosf(threadIdx.x * 2e-3f), vi = sinf(threadIdx.x * 2e-3f);
  for (int it = 0; it < iters; it += 2) {
    u64 A = pk(1.f, 0.f), B = pk(wr, wi), A2 = pk(1.f, 0.f), B2 = pk(vr, vi);
    const u64 C = pk(2.f * wr, 2.f * wr), C2 = pk(2.f * vr, 2.f * vr);
#pragma unroll
    for (int j = 0; j < M; j++) {
      if (j) {
        u64 N = ffma2(B, C, neg2(A)); A = B; B = N;
        u64 N2 = ffma2(B2, C2, neg2(A2)); A2 = B2; B2 = N2;
      }
      S[j] = fadd2(fadd2(S[j], B), B2);
    }
    wr += 1e-7f; wi -= 1e-7f; vr -= 1e-7f; vi += 1e-7f;
  }
  float s = 0; for (int j = 0; j < M; j++) { float2 v = upk(S[j]); s += v.x + v.y; }
  if (s == 1234.5f) g_sink[0] = s;
}

// pairs (v_{k+1}, v_{k+17}), k = 0..15, of one photon; X = re chain, Y = im chain
template <int NT>
__global__ void __launch_bounds__(NT) k_jsplit(float* out, int iters) {
  constexpr int H = 16;
  u64 SR[H], SI[H];
#pragma unroll
  for (int k = 0; k < H; k++) SR[k] = SI[k] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  float ar = cosf(threadIdx.x * 3e-3f), ai = sinf(threadIdx.x * 3e-3f);
  for (int it = 0; it < iters; it++) {
    const float c2 = 2.f * wr;
    const u64 C = pk(c2, c2);
    u64 Xa = pk(1.f, ar), Xb = pk(wr, ai), Ya = pk(0.f, ai), Yb = pk(wi, ar);  // (v_0, v_16), (v_1, v_17)
#pragma unroll
    for (int k = 0; k < H; k++) {
      if (k) {
        u64 Xn = ffma2(C, Xb, neg2(Xa)); Xa = Xb; Xb = Xn;
        u64 Yn = ffma2(C, Yb, neg2(Ya)); Ya = Yb; Yb = Yn;
      }
      SR[k] = fadd2(SR[k], Xb);
      SI[k] = fadd2(SI[k], Yb);
    }
    wr += 1e-7f; wi -= 1e-7f; ar += 1e-7f; ai -= 1e-7f;
  }
  float s = 0; for (int k = 0; k < H; k++) { float2 v = upk(SR[k]), u = upk(SI[k]); s += v.x + v.y + u.x + u.y; }
  if (s == 1234.5f) g_sink[0] = s;
}

// jsplit with two photons interleaved (ILP 2, separate chains, shared accumulators)
template <int NT>
__global__ void __launch_bounds__(NT) k_jsplit2(float* out, int iters) {
  constexpr int H = 16;
  u64 SR[H], SI[H];
#pragma unroll
  for (int k = 0; k < H; k++) SR[k] = SI[k] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  float vr = cosf(threadIdx.x * 2e-3f), vi = sinf(threadIdx.x * 2e-3f);
  float ar = cosf(threadIdx.x * 3e-3f), ai = sinf(threadIdx.x * 3e-3f);
  for (int it = 0; it < iters; it += 2) {
    const u64 C = pk(2.f * wr, 2.f * wr), D = pk(2.f * vr, 2.f * vr);
    u64 Xa = pk(1.f, ar), Xb = pk(wr, ai), Ya = pk(0.f, ai), Yb = pk(wi, ar);
    u64 Pa = pk(1.f, ai), Pb = pk(vr, ar), Qa = pk(0.f, ar), Qb = pk(vi, ai);
#pragma unroll
    for (int k = 0; k < H; k++) {
      if (k) {
        u64 Xn = ffma2(C, Xb, neg2(Xa)); Xa = Xb; Xb = Xn;
        u64 Yn = ffma2(C, Yb, neg2(Ya)); Ya = Yb; Yb = Yn;
        u64 Pn = ffma2(D, Pb, neg2(Pa)); Pa = Pb; Pb = Pn;
        u64 Qn = ffma2(D, Qb, neg2(Qa)); Qa = Qb; Qb = Qn;
      }
      SR[k] = fadd2(fadd2(SR[k], Xb), Pb);
      SI[k] = fadd2(fadd2(SI[k], Yb), Qb);
    }
    wr += 1e-7f; wi -= 1e-7f; vr -= 1e-7f; vi += 1e-7f; ar += 1e-7f; ai -= 1e-7f;
  }
  float s = 0; for (int k = 0; k < H; k++) { float2 v = upk(SR[k]), u = upk(SI[k]); s += v.x + v.y + u.x + u.y; }
  if (s == 1234.5f) g_sink[0] = s;
}

// two-slot: pairs (photon p, photon q) of one component, coefficient pair (c_p, c_q)
template <int NT, int M>
__global__ void __launch_bounds__(NT) k_twoslot(float* out, int iters) {
  u64 SX[M], SY[M];
#pragma unroll
  for (int j = 0; j < M; j++) SX[j] = SY[j] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  float vr = cosf(threadIdx.x * 2e-3f), vi = sinf(threadIdx.x * 2e-3f);
  for (int it = 0; it < iters; it += 2) {
    const u64 C = pk(2.f * wr, 2.f * vr);
    u64 Xa = pk(1.f, 1.f), Xb = pk(wr, vr), Ya = pk(0.f, 0.f), Yb = pk(wi, vi);
#pragma unroll
    for (int j = 0; j < M; j++) {
      if (j) {
        u64 Xn = ffma2(C, Xb, neg2(Xa)); Xa = Xb; Xb = Xn;
        u64 Yn = ffma2(C, Yb, neg2(Ya)); Ya = Yb; Yb = Yn;
      }
      SX[j] = fadd2(SX[j], Xb);
      SY[j] = fadd2(SY[j], Yb);
    }
    wr += 1e-7f; wi -= 1e-7f; vr -= 1e-7f; vi += 1e-7f;
  }
  float s = 0; for (int j = 0; j < M; j++) { float2 v = upk(SX[j]), u = upk(SY[j]); s += v.x + v.y + u.x + u.y; }
  if (s == 1234.5f) g_sink[0] = s;
}

// scalar FFMA chains, accumulate (x_j, x_{j+1}) pairs
template <int NT>
__global__ void __launch_bounds__(NT) k_srpa(float* out, int iters) {
  constexpr int M = 32;
  u64 SR[M / 2], SI[M / 2];
#pragma unroll
  for (int k = 0; k < M / 2; k++) SR[k] = SI[k] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  for (int it = 0; it < iters; it++) {
    const float c2 = 2.f * wr;
    float x0 = 1.f, x1 = wr, y0 = 0.f, y1 = wi;
#pragma unroll
    for (int k = 0; k < M / 2; k++) {
      // terms j = 2k+1, 2k+2
      float xa = x1, ya = y1;
      float xb = fmaf(c2, x1, -x0), yb = fmaf(c2, y1, -y0);
      SR[k] = fadd2(SR[k], pk(xa, xb));
      SI[k] = fadd2(SI[k], pk(ya, yb));
      x0 = xb; y0 = yb;
      x1 = fmaf(c2, xb, -xa); y1 = fmaf(c2, yb, -ya);
    }
    wr += 1e-7f; wi -= 1e-7f;
  }
  float s = 0; for (int k = 0; k < M / 2; k++) { float2 v = upk(SR[k]), u = upk(SI[k]); s += v.x + v.y + u.x + u.y; }
  if (s == 1234.5f) g_sink[0] = s;
}


// cheb2q fed from a shared-memory phase table (random bins, like the kernel): per photon one
// LDS.64 + seeds; NB blocks of 256 per SM (occupancy control)
template <int NT>
__global__ void __launch_bounds__(NT, 2) k_cheb2q_tab(float* out, int iters) {
  constexpr int M = 32;
  __shared__ float2 tab[4096];  // (the kernel's table is 64 KB dynamic; 32 KB static here, same access pattern)
  for (int i = threadIdx.x; i < 4096; i += NT) tab[i] = make_float2(cosf(i * 1.53e-3f), sinf(i * 1.53e-3f));
  __syncthreads();
  u64 S[M];
#pragma unroll
  for (int j = 0; j < M; j++) S[j] = 0;
  uint32_t x = threadIdx.x * 2654435761u, y = threadIdx.x * 40503u + 17u;
  for (int it = 0; it < iters; it += 2) {
    x = x * 1664525u + 1013904223u;
    y = y * 22695477u + 1u;
    const float2 w = tab[x >> 20], v = tab[y >> 20];
    u64 A = pk(1.f, 0.f), B = pk(w.x, w.y), A2 = pk(1.f, 0.f), B2 = pk(v.x, v.y);
    const u64 C = pk(2.f * w.x, 2.f * w.x), C2 = pk(2.f * v.x, 2.f * v.x);
#pragma unroll
    for (int j = 0; j < M; j++) {
      if (j) {
        u64 N = ffma2(B, C, neg2(A)); A = B; B = N;
        u64 N2 = ffma2(B2, C2, neg2(A2)); A2 = B2; B2 = N2;
      }
      S[j] = fadd2(fadd2(S[j], B), B2);
    }
  }
  float s = 0; for (int j = 0; j < M; j++) { float2 v = upk(S[j]); s += v.x + v.y; }
  if (s == 1234.5f) g_sink[0] = s;
}
template <int NT>
__global__ void __launch_bounds__(NT, 2) k_cheb2q_lb2(float* out, int iters) {
  constexpr int M = 32;
  u64 S[M];
#pragma unroll
  for (int j = 0; j < M; j++) S[j] = 0;
  float wr = cosf(threadIdx.x * 1e-3f), wi = sinf(threadIdx.x * 1e-3f);
  float vr = cosf(threadIdx.x * 2e-3f), vi = sinf(threadIdx.x * 2e-3f);
  for (int it = 0; it < iters; it += 2) {
    u64 A = pk(1.f, 0.f), B = pk(wr, wi), A2 = pk(1.f, 0.f), B2 = pk(vr, vi);
    const u64 C = pk(2.f * wr, 2.f * wr), C2 = pk(2.f * vr, 2.f * vr);
#pragma unroll
    for (int j = 0; j < M; j++) {
      if (j) {
        u64 N = ffma2(B, C, neg2(A)); A = B; B = N;
        u64 N2 = ffma2(B2, C2, neg2(A2)); A2 = B2; B2 = N2;
      }
      S[j] = fadd2(fadd2(S[j], B), B2);
    }
    wr += 1e-7f; wi -= 1e-7f; vr -= 1e-7f; vi += 1e-7f;
  }
  float s = 0; for (int j = 0; j < M; j++) { float2 v = upk(S[j]); s += v.x + v.y; }
  if (s == 1234.5f) g_sink[0] = s;
}

typedef void (*kfn)(float*, int);
static void run(const char* name, kfn f, int bs, int iters, double terms_per_iter, int nsm, float* out) {
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, bs, 0));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, f));
  const int grid = nsm * per_sm;
  f<<<grid, bs>>>(out, 8);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; r++) {
    cudaEventRecord(e0);
    f<<<grid, bs>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double terms = terms_per_iter * iters * (double)bs * grid;
  const double per_clk = terms / (best * 1e-3) / (nsm * 1.965e9);
  printf("{\"test\":\"%s\",\"threads\":%d,\"regs\":%d,\"blocks_per_sm\":%d,\"terms_per_clk_per_sm\":%.2f,"
         "\"frac_of_fp32_roofline\":%.3f,\"ms\":%.3f}\n", name, bs, fa.numRegs, per_sm, per_clk, per_clk / 32.0, best);
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  float* out; CK(cudaMalloc(&out, 1024));
  const int IT = 2000;
  run("cheb2q_tab_256x2", k_cheb2q_tab<256>, 256, IT, 32, nsm, out);
  run("cheb2q_lb2_256x2", k_cheb2q_lb2<256>, 256, IT, 32, nsm, out);
  run("cheb1_256", k_cheb1<256>, 256, IT, 32, nsm, out);
  run("cheb1_512", k_cheb1<512>, 512, IT, 32, nsm, out);
  run("cheb2p_256", k_cheb2p<256>, 256, IT, 32, nsm, out);
  run("cheb2p_512", k_cheb2p<512>, 512, IT, 32, nsm, out);
  run("cheb2q_256", k_cheb2q<256>, 256, IT, 32, nsm, out);
  run("jsplit_256", k_jsplit<256>, 256, IT, 32, nsm, out);
  run("jsplit_512", k_jsplit<512>, 512, IT, 32, nsm, out);
  run("jsplit_1024", k_jsplit<1024>, 1024, IT, 32, nsm, out);
  run("jsplit2_256", k_jsplit2<256>, 256, IT, 32, nsm, out);
  run("jsplit2_512", k_jsplit2<512>, 512, IT, 32, nsm, out);
  run("twoslot16_256", k_twoslot<256, 16>, 256, IT, 16, nsm, out);
  run("twoslot16_512", k_twoslot<512, 16>, 512, IT, 16, nsm, out);
  run("twoslot32_256", k_twoslot<256, 32>, 256, IT, 32, nsm, out);
  run("srpa_256", k_srpa<256>, 256, IT, 32, nsm, out);
  run("srpa_512", k_srpa<512>, 512, IT, 32, nsm, out);
  return 0;
}
