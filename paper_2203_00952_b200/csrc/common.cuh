// Shared device helpers for the SRT3D sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace srt3d {

typedef unsigned long long u64;

// ---- packed fp32x2 arithmetic (sm_100a FFMA2 / FMUL2 / FADD2) -------------
// A u64 holds (lo, hi) = (re, im).  ptxas folds the scalar broadcasts built
// with pk(s, s) into the .F32 operand form, so no MOVs are emitted.
__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo_of(u64 v) {
  float a, b;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi_of(u64 v) {
  float a, b;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// -v (ptxas folds the negation into the consuming FFMA2/FADD2 operand).
__device__ __forceinline__ u64 neg2(u64 v) { return pk(-lo_of(v), -hi_of(v)); }

// Complex multiply p * w with packed ops: (pr,pr)*(wr,wi) + (pi,pi)*(-wi,wr).
// W = (wr, wi), Wn = (-wi, wr).  2 instructions, 4 FP32 lane-ops.
__device__ __forceinline__ u64 cmul2(u64 p, u64 W, u64 Wn) {
  return ffma2(pk(hi_of(p), hi_of(p)), Wn, fmul2(pk(lo_of(p), lo_of(p)), W));
}

// ---- exact integer phase index (PAPER.md:61 with omega_j = 2 pi j / T) -----
// (n mod T) for n < 2^23 without an integer division: fp32 quotient estimate
// (n is exact in fp32, q is off by at most one) corrected by one step.
__device__ __forceinline__ uint32_t mod_small(uint32_t n, uint32_t T, float invT) {
  uint32_t q = __float2uint_rz(__uint2float_rz(n) * invT);
  int r = (int)n - (int)(q * T);
  if (r < 0) r += (int)T;
  if (r >= (int)T) r -= (int)T;
  return (uint32_t)r;
}
// r = (j * x) mod T for x < T <= 65536, j <= 64 (j*x < 2^22): the index of
// exp(i omega_j x) in the exact phase table.  Used by every sketch path for
// its anchors and by srt3d_debug_phase_index (bit-exactness test).
__device__ __forceinline__ uint32_t phase_index(uint32_t x, uint32_t j, uint32_t T, float invT) {
  return mod_small(j * x, T, invT);
}

// ---- fixed-point phase of a real depth (expected sketch / gradient) --------
// q = round(frac(t / T) * 2^32) as uint32: t/T in revolutions, 32-bit fixed
// point.  j*q (mod 2^32) is then the exact phase of omega_j * t up to the
// 2^-33 revolution quantisation of q, for any j (no fp32 range-reduction
// error even when j*t is large).
__device__ __forceinline__ uint32_t phase_q32(float t, double invT) {
  double r = (double)t * invT;  // revolutions, relative error ~1e-16
  r -= floor(r);                // frac in [0, 1)
  return (uint32_t)(unsigned long long)__double2ll_rn(r * 4294967296.0);  // 2^32 wraps to 0
}
// exp(i * 2 pi * q / 2^32) with q interpreted as a signed half-open
// revolution in [-1/2, 1/2): sincospif on a = q * 2^-31 in [-1, 1).
// (A 256-entry table + residual polynomial variant, tools/gen_phase_tab.py,
// was as accurate but slower in the kernel: the dependent global table load
// sits on the anchor's critical path.)
// The 32-bit phase is split into its top 24 bits (exact as an fp32 argument) and
// the 8 low bits, applied as a first-order rotation by d = pi ql 2^-31 <= 3.7e-7
// rad (the d^2/2 term is below 7e-14): converting all 32 bits to fp32 would round
// the angle by up to 1.9e-7 rad, an error the recurrences built on this anchor
// multiply by their length (round 2: A12's floor was exceeded by up to 1.4x at
// m = 32 for T not a power of two, tools/a12_probe.py).  When the low bits are
// zero (e.g. t / T with T a power of two) the result is bitwise sincospif's.
__device__ __forceinline__ float2 phasor_q32(uint32_t q) {
  const int32_t qi = (int32_t)q;
  const int32_t qh = qi & ~0xFF, ql = qi - qh;  // qh: 24 significant bits
  const float a = (float)qh * 4.656612873077392578125e-10f;  // 2^-31, exact
  float s, c;
  sincospif(a, &s, &c);
  const float d = (float)ql * 1.4629180792671596e-9f;  // pi 2^-31
  return make_float2(fmaf(-s, d, c), fmaf(c, d, s));
}

}  // namespace srt3d
