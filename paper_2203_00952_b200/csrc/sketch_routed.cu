// K1 — class-routed Chebyshev sketch, Eq. (3):
//
//   z[i][j-1] = (1/n_i) sum_p exp(i 2 pi j x_p / T),  j = 1 .. M  (one pass, M <= 32)
//
// The cheapest phasor recurrence on sm_100a is the Chebyshev one: both
// components of v_j = e^{i j phi} obey v_j = 2 cos(phi) v_{j-1} - v_{j-2},
// ONE FFMA2 per (photon, j) beside the FADD2 that accumulates it (the complex
// power needs FMUL2 + FFMA2: 3 packed instructions per term instead of 2).
// In fp32 the recurrence is accurate only where |sin phi| is not small, so
// each photon runs in one of two frames:
//   frame A: phi = theta,         accurate iff |sin theta| >= tau,
//   frame B: phi = theta + pi/2,  accurate iff |cos theta| >= tau
//            (e^{i j phi} = i^j e^{i j theta}: the frame-B sums are rotated
//            back by (-i)^j once per fold),
// tau = 0.2: worst phasor error 4.9e-6 for j <= 32 at every T tested
// (tools/sim_cheb_tau.c), inside the 1e-5 sketch tolerance even when every
// photon of a pixel sits in one worst-case bin.
//
// A pixel is owned by a PAIR of lanes: the even lane's accumulators are in
// frame A, the odd lane's in frame B.  Each round both lanes load 8 photons
// (one 16-byte vector each), classify them from the exact table entry
// e^{i theta} = tab[x], swap masks with one shuffle, and decide per slot:
//   keep  — A-lane runs its own photon, B-lane its own;
//   swap  — they exchange photons (the x values come with the same shuffle);
//   clash — both photons need the same frame (3.3 % of slots for uniform
//           photons): that frame's lane runs its photon, the other photon is
//           appended to a per-pair spill list of that frame, run later.
// So each lane runs exactly 8 photon slots per round (a clash leaves one
// empty slot) through the class-uniform body, two photons at a time, no
// divergence.  A warp runs 16 pixels (one per pair) in lockstep; every ~128
// photon slots per lane, and at the end of the pixels, the spill lists are
// drained and the partial sums folded (frame B rotated back, pair shuffle
// reduce) into per-lane shared-memory partials, warp-uniformly.  The order of
// every sum is fixed, so results are bitwise reproducible.
#include <cstdint>
#include <utility>

#include "sketch_impl.cuh"

namespace srt3d {

constexpr float RT_TAU = 0.2f;            // frame accuracy threshold (tools/sim_cheb_tau.c: 4.9e-6; 0.25: 4.1e-6
                                          // but 5.2 % clash slots instead of 3.3 %)
constexpr int RT_THREADS = 512;           // CTA size: one CTA per SM (shared memory), 16 warps
constexpr int RT_FOLD_ROUNDS = 16;        // rounds between folds: <= 128 photon slots per lane per partial
constexpr int RT_SPILL_CAP = 32;          // spill-list entries per lane (uint16 bins)

struct RtBody {
  template <int M, int J>
  __device__ __forceinline__ static void term(u64 (&acc)[M], u64& Ap, u64& Bp, u64& Aq, u64& Bq, u64 Cp, u64 Cq) {
    if constexpr (J > 0) {
      const u64 Np = ffma2(Bp, Cp, neg2(Ap));
      const u64 Nq = ffma2(Bq, Cq, neg2(Aq));
      Ap = Bp;
      Bp = Np;
      Aq = Bq;
      Bq = Nq;
    }
    acc[J] = fadd2(acc[J], fadd2(Bp, Bq));
  }
  template <int M, int... J>
  __device__ __forceinline__ static void terms(std::integer_sequence<int, J...>, u64 (&acc)[M], u64& Ap, u64& Bp,
                                               u64& Aq, u64& Bq, u64 Cp, u64 Cq) {
    (term<M, J>(acc, Ap, Bp, Aq, Bq, Cp, Cq), ...);
  }
  // Two photons with base phasors w, u in this lane's frame.  An absent photon
  // reads the zero table entry (w = 0, so the coefficient is 0 too) and its
  // v_0 seed is gated by the valid flag: all its terms are exactly 0.
  template <int M>
  __device__ __forceinline__ static void pair(u64 (&acc)[M], float2 w, bool wv, float2 u, bool uv) {
    u64 Ap = pk(wv ? 1.f : 0.f, 0.f), Bp = pk(w.x, w.y);
    u64 Aq = pk(uv ? 1.f : 0.f, 0.f), Bq = pk(u.x, u.y);
    const float cp = 2.f * w.x, cq = 2.f * u.x;
    terms(std::make_integer_sequence<int, M>{}, acc, Ap, Bp, Aq, Bq, pk(cp, cp), pk(cq, cq));
  }
};

__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

// Frame B -> frame A for term J (j = J + 1): multiply by (-i)^j on the B lane.
template <int J>
__device__ __forceinline__ void rt_unrotate(float& re, float& im, bool fb) {
  constexpr int r = (J + 1) & 3;
  if constexpr (r == 1) {  // (-i)(a + ib) = (b, -a)
    const float a = re, b = im;
    re = fb ? b : a;
    im = fb ? -a : b;
  } else if constexpr (r == 2) {
    re = fb ? -re : re;
    im = fb ? -im : im;
  } else if constexpr (r == 3) {  // (+i)(a + ib) = (-b, a)
    const float a = re, b = im;
    re = fb ? -b : a;
    im = fb ? a : b;
  }
}

template <int NV, int... J>
__device__ __forceinline__ void rt_unrotate_all(float (&f)[NV], bool fb, std::integer_sequence<int, J...>) {
  (rt_unrotate<J>(f[2 * J], f[2 * J + 1], fb), ...);
}

// Shared memory of the routed kernel for T (T % 4 == 0) (cls static, the rest dynamic):
//   ptab[T + T/4 + 1]  e^{i 2 pi x / T} for x < T + T/4 (the wrap-around copy lets
//                      a frame-B lane read e^{i(theta + pi/2)} = ptab[x + T/4] with
//                      no index arithmetic: its table base is ptab + T/4), and
//                      ptab[T + T/4] = 0: the absent photon (index T + T/4 in frame A,
//                      T in frame B)
//   part[M][RT_THREADS] per-lane fp32 partial sums (transposed: conflict-free)
//   spill[RT_THREADS][RT_SPILL_CAP] uint16 per-lane spill lists
//   cls[T + 1]         class byte of bin x: bit 0 frame A accurate (|sin| >= tau),
//                      bit 1 frame B accurate (|cos| >= tau); cls[T] = 0 (no photon)
__host__ __device__ constexpr size_t rt_tab_entries(uint32_t T) { return ((size_t)T + T / 4 + 2) & ~(size_t)1; }
size_t sketch_routed_smem(uint32_t T, int M) {
  return sizeof(float2) * rt_tab_entries(T) + sizeof(float) * (size_t)RT_THREADS * M +
         sizeof(uint16_t) * (size_t)RT_THREADS * RT_SPILL_CAP;
}

constexpr int RT_WIN = 128;         // pixels per sorted window (4 per lane)
constexpr uint32_t RT_PIX_W = 16;   // per-pixel weight (in photons) of the warp split: the head round

// Smallest p in [0, npix] with weight(p) = (offsets[p] - offsets[0]) + RT_PIX_W * p >= target,
// by a warp-cooperative 32-ary search (the weight is nondecreasing for a valid CSR; for a
// malformed one the result is still in range).  Warp-uniform.
__device__ __forceinline__ long long rt_split(const uint32_t* __restrict__ off, long long npix, unsigned long long target,
                                             int lane) {
  const uint32_t base = off[0];
  long long lo = 0, hi = npix;  // the answer lies in [lo, hi]
  while (hi - lo > 32) {
    const long long q = lo + ((hi - lo) * (lane + 1)) / 32;  // lane 31 probes hi
    const bool ge = (unsigned long long)(off[q] - base) + (unsigned long long)RT_PIX_W * q >= target;
    const uint32_t b = __ballot_sync(0xffffffffu, ge) | 0x80000000u;
    const int f = __ffs(b) - 1;
    const long long qf = __shfl_sync(0xffffffffu, q, f);
    const long long qp = __shfl_sync(0xffffffffu, q, f > 0 ? f - 1 : 0);
    lo = f > 0 ? qp + 1 : lo;
    hi = qf;
  }
  const long long q = lo + lane;
  const bool ge = q >= hi || (unsigned long long)(off[q] - base) + (unsigned long long)RT_PIX_W * q >= target;
  const int f = __ffs(__ballot_sync(0xffffffffu, ge)) - 1;  // lane hi - lo <= 32... lane 31 at most
  return f < 0 ? hi : lo + f;
}

// Bitonic sort of the warp's 128 keys (key[i] at position 32 i + lane), descending.
__device__ __forceinline__ void rt_sort128(uint32_t (&key)[4], int lane) {
#pragma unroll
  for (int k = 2; k <= RT_WIN; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jj = j >> 5;
#pragma unroll
        for (int i = 0; i < 4; i++) {
          if (i & jj) continue;
          const bool up = ((32 * i) & k) == 0;  // this block sorts descending (up) or ascending
          const uint32_t a0 = key[i], a1 = key[i | jj];
          key[i] = up ? max(a0, a1) : min(a0, a1);
          key[i | jj] = up ? min(a0, a1) : max(a0, a1);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, key[i], j);
          const bool up = ((32 * i + lane) & k) == 0, lower = (lane & j) == 0;
          key[i] = (up == lower) ? max(key[i], o) : min(key[i], o);
        }
      }
    }
  }
}

template <int M>
__global__ void __launch_bounds__(RT_THREADS, 1) sketch_routed_kernel(SketchArgs a) {
  extern __shared__ float2 rt_smem[];
  if (sketch_regime_skip(a, M)) return;  // another candidate launch of this pass does the work
  constexpr int NV = 2 * M;              // floats per pixel
  constexpr int HV = M;                  // floats per lane after the pair reduce (NV / 2)
  const uint32_t T = a.T, Q = T / 4;
  // cls is a static array: its byte address is the photon index plus an immediate
  __shared__ uint8_t cls[RT_MAX_T + 1];
  float2* ptab = rt_smem;
  float* part = reinterpret_cast<float*>(ptab + rt_tab_entries(T));                // [HV][RT_THREADS]
  uint16_t* spill = reinterpret_cast<uint16_t*>(part + (size_t)RT_THREADS * HV);   // [RT_THREADS][CAP]
  {  // tables: fp64 sincospi on the centred index, rounded once; classes from the fp32 values
    const double sc = 2.0 / (double)T;
    for (uint32_t r = threadIdx.x; r < T + Q + 1; r += RT_THREADS) {
      const uint32_t x = r < T ? r : r - T;
      const int rc = (2u * x > T) ? (int)x - (int)T : (int)x;
      double sn, cs;
      sincospi(sc * (double)rc, &sn, &cs);
      const float2 w = make_float2((float)cs, (float)sn);
      ptab[r] = r == T + Q ? make_float2(0.f, 0.f) : w;  // [T + Q]: the absent-photon entry of both frames
      if (r < T) cls[r] = (uint8_t)((fabsf(w.y) >= RT_TAU ? 1u : 0u) | (fabsf(w.x) >= RT_TAU ? 2u : 0u));
    }
    if (threadIdx.x == 0) cls[T] = 0;
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const bool fb = lane & 1;                  // frame-B lane (odd), frame-A lane (even)
  const int pr = lane >> 1;                  // pair index in the warp = pixel index in the tile
  // my table as a shared-window byte address (frame B: e^{i(theta + pi/2)} = ptab[x + T/4]) and
  // my absent-photon index: ptab[T + T/4] = 0 in both frames
  const uint32_t mytab = (uint32_t)__cvta_generic_to_shared(ptab) + (fb ? 8u * Q : 0u);
  const uint32_t xnone = fb ? T : T + Q;
  float* mypart = part + threadIdx.x;        // element i at mypart[i * RT_THREADS]
  // spill list of MY frame (photons the partner could not run; the partner writes it)
  const uint16_t* myspill = spill + (size_t)threadIdx.x * RT_SPILL_CAP;
  uint16_t* ptspill = spill + (size_t)(threadIdx.x ^ 1) * RT_SPILL_CAP;  // the partner's frame list (I write)
  const long long warp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const uint32_t off0 = (uint32_t)(((uintptr_t)a.bins >> 1) & 7u);
  const uint4* __restrict__ vb = reinterpret_cast<const uint4*>(a.bins - off0);
  const uint16_t* __restrict__ bins = a.bins;
  const uint32_t TT = T | (T << 16);

  u64 acc[M];
#pragma unroll
  for (int j = 0; j < M; j++) acc[j] = 0ull;
  int nsp_part = 0;  // entries I wrote into the partner's frame list since the last drain

  // Drain the spill lists (each lane runs its frame's list, two photons per step) and
  // fold acc into the per-lane partials: frame B rotated back, pair reduce (lane A keeps
  // floats [0, M), lane B [M, 2M)).  Called warp-uniformly; fixed order.
  auto drain_and_fold = [&]() {
    __syncwarp();  // the partner's spill stores are visible
    const int n = __shfl_xor_sync(0xffffffffu, nsp_part, 1);
    for (int k = 0; k < n; k += 2) {
      const bool v1 = k + 1 < n;
      const float2 e0 = lds_f2(mytab + 8u * myspill[k]);
      const float2 e1 = lds_f2(mytab + 8u * (v1 ? (uint32_t)myspill[k + 1] : xnone));
      RtBody::pair<M>(acc, e0, true, e1, v1);
    }
    nsp_part = 0;
    float f[NV];
#pragma unroll
    for (int j = 0; j < M; j++) {
      f[2 * j] = lo_of(acc[j]);
      f[2 * j + 1] = hi_of(acc[j]);
      acc[j] = 0ull;
    }
    rt_unrotate_all(f, fb, std::make_integer_sequence<int, M>{});
#pragma unroll
    for (int i = 0; i < HV; i++) {
      const float send = fb ? f[i] : f[i + HV];
      const float keep = fb ? f[i + HV] : f[i];
      mypart[i * RT_THREADS] += keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
    __syncwarp();  // the lists may be refilled
  };

  // This warp's pixels: a contiguous range of equal weight (photons + RT_PIX_W per pixel), so
  // warps finish together whatever the spatial photon distribution.  The range is taken in
  // windows of up to 128 pixels sorted by photon count, and each 16-pixel tile (one pixel per
  // lane pair, run in lockstep) takes 16 consecutive ranks: lanes of a tile run for nearly the
  // same number of rounds.
  long long p0, p1;
  {
    const unsigned long long total =
        (unsigned long long)(a.offsets[a.npix] - a.offsets[0]) + (unsigned long long)RT_PIX_W * a.npix;
    p0 = rt_split(a.offsets, a.npix, total * warp0 / nwarps, lane);
    p1 = rt_split(a.offsets, a.npix, total * (warp0 + 1) / nwarps, lane);
  }
  for (long long wb = p0; wb < p1; wb += RT_WIN) {
    const int W = (int)min((long long)RT_WIN, p1 - wb);
    uint32_t key[4];  // (count + 1) << 7 | local index; 0 = no pixel (sorts last)
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int li = 32 * i + lane;
      key[i] = 0;
      if (li < W) {
        const uint32_t b0 = a.offsets[wb + li], b1 = a.offsets[wb + li + 1];
        const uint32_t c = b1 > b0 ? min(b1 - b0, (1u << 24) - 2u) : 0u;
        key[i] = ((c + 1u) << 7) | (uint32_t)li;
      }
    }
    rt_sort128(key, lane);
    const int ntile = (W + 15) >> 4;
    for (int tl = 0; tl < ntile; tl++) {
    // rank 16 tl + pr sits at position 32 (tl >> 1) + 16 (tl & 1) + pr
    const uint32_t kw = tl < 2 ? key[0] : (tl < 4 ? key[1] : (tl < 6 ? key[2] : key[3]));
    const uint32_t kt = __shfl_sync(0xffffffffu, kw, ((tl & 1) << 4) | pr);
    const int rank = 16 * tl + pr;
    const bool valid = rank < W && kt != 0;
    const long long pix = wb + (kt & 127u);
    uint32_t beg = 0, end = 0;
    if (valid) {
      beg = a.offsets[pix];
      end = a.offsets[pix + 1];
    }
    if (end < beg) end = beg;  // malformed CSR: treat as empty (never read out of range)
    // slot space s = photon index + off0 (16-byte aligned when s % 8 == 0), 64-bit: s may reach 2^32 + 7
    const unsigned long long asb = ((unsigned long long)beg + off0 + 7u) & ~7ull;
    const unsigned long long ase = ((unsigned long long)end + off0) & ~7ull;
    uint32_t hend = end, tbeg = end;
    long long cb = 0, ce = 0;  // 16-byte chunk indices
    if (asb < ase) {
      hend = (uint32_t)(asb - off0);
      tbeg = (uint32_t)(ase - off0);
      cb = (long long)(asb >> 3);
      ce = (long long)(ase >> 3);
    }
    const int nh = (int)(hend - beg), nht = nh + (int)(end - tbeg);
    // round 0: head + tail scalars (< 16: slot i of lane l takes scalar 2i + l);
    // rounds 1..: one 16-byte chunk per lane, the pair's chunks cb + 2(r-1) + l.
    // An empty slot holds 0xffff, clamped to T: class 0, no photon.
    int nr = 1 + (int)((ce - cb + 1) >> 1);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) nr = max(nr, __shfl_xor_sync(0xffffffffu, nr, d));
#pragma unroll
    for (int i = 0; i < HV; i++) mypart[i * RT_THREADS] = 0.f;

    uint32_t hv[8];  // round 0: the scalars
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const int idx = 2 * i + (int)fb;
      hv[i] = idx < nht ? (uint32_t)bins[idx < nh ? (size_t)beg + idx : (size_t)tbeg + (idx - nh)] : 0xffffu;
    }
    uint32_t nw[4];  // the next round's photons (prefetched)
#pragma unroll
    for (int q = 0; q < 4; q++) nw[q] = hv[2 * q] | (hv[2 * q + 1] << 16);
    for (int r = 0; r < nr; r++) {
      uint32_t wv[4];
#pragma unroll
      for (int q = 0; q < 4; q++) wv[q] = __vminu2(nw[q], TT);  // bins >= T (or empty) -> T
      {  // prefetch round r + 1
        const long long cl = cb + 2ll * r + (long long)fb;
        if (cl < ce) {
          const uint4 v = __ldg(vb + cl);
          nw[0] = v.x;
          nw[1] = v.y;
          nw[2] = v.z;
          nw[3] = v.w;
        } else {
          nw[0] = nw[1] = nw[2] = nw[3] = 0xffffffffu;
        }
      }
      // ---- class codes of my 8 photons: bits (2i, 2i + 1) of cc = (frame A, frame B) accurate
      uint32_t cc = 0;
#pragma unroll
      for (int i = 0; i < 8; i++) cc += (uint32_t)cls[(wv[i >> 1] >> (16 * (i & 1))) & 0xffffu] << (2 * i);
      // ---- exchange with the partner: its photons and class codes
      uint32_t pw[4];
#pragma unroll
      for (int q = 0; q < 4; q++) pw[q] = __shfl_xor_sync(0xffffffffu, wv[q], 1);
      const uint32_t pc = __shfl_xor_sync(0xffffffffu, cc, 1);
      // P = the A lane's photon of a slot, Q = the B lane's; masks hold slot i at bit 2i
      constexpr uint32_t EV = 0x5555u;
      const uint32_t Pc = fb ? pc : cc, Qc = fb ? cc : pc;
      const uint32_t aP = Pc & EV, bP = (Pc >> 1) & EV, aQ = Qc & EV, bQ = (Qc >> 1) & EV;
      const uint32_t vP = aP | bP, vQ = aQ | bQ;
      // keep: each lane runs its own photon; swap: exchange; clash: both need one frame
      const uint32_t keep = (aP & bQ) | (aP & ~vQ) | (bQ & ~vP);
      const uint32_t swap = ~keep & ((aQ & bP) | (vP & ~vQ) | (vQ & ~vP));
      const uint32_t clash = vP & vQ & ~keep & ~swap;
      const uint32_t clashA = clash & aP;   // both frame-A only: A runs P, Q -> A's spill list
      const uint32_t clashB = clash & ~aP;  // both frame-B only: B runs Q, P -> B's spill list
      // my slot: own photon if keep or a clash in my frame; the partner's if swap (and it has one)
      const uint32_t own = fb ? ((keep & vQ) | clashB) : ((keep & vP) | clashA);
      const uint32_t other = swap & (fb ? vP : vQ);
      uint32_t spl = fb ? clashA : clashB;  // my own photon goes to the partner's frame list
      while (spl) {  // rare (~5 % of slots): one iteration per spilled photon
        const int i = (__ffs(spl) - 1) >> 1;
        spl &= spl - 1;
        const uint32_t w = i >= 4 ? (i >= 6 ? wv[3] : wv[2]) : (i >= 2 ? wv[1] : wv[0]);
        ptspill[nsp_part++] = (uint16_t)(w >> (16 * (i & 1)));
      }
      // ---- the 8 slots through the class-uniform body, two per step; an empty slot
      // reads the zero entry
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const bool s0 = (other >> (2 * i)) & 1u, s1 = (other >> (2 * i + 2)) & 1u;
        const bool o0 = (own >> (2 * i)) & 1u, o1 = (own >> (2 * i + 2)) & 1u;
        const uint32_t wq = wv[i >> 1], pq = pw[i >> 1];
        const uint32_t x0 = s0 ? (pq & 0xffffu) : (o0 ? (wq & 0xffffu) : xnone);
        const uint32_t x1 = s1 ? (pq >> 16) : (o1 ? (wq >> 16) : xnone);
        const float2 e0 = lds_f2(mytab + 8u * x0);
        const float2 e1 = lds_f2(mytab + 8u * x1);
        RtBody::pair<M>(acc, e0, s0 || o0, e1, s1 || o1);
      }
      // ---- warp-uniform drain + fold: every RT_FOLD_ROUNDS rounds, when a spill list
      // could overflow next round, and at the end of the tile
      const bool full = __any_sync(0xffffffffu, nsp_part > RT_SPILL_CAP - 8);
      if (r == nr - 1 || full || (r + 1) % RT_FOLD_ROUNDS == 0) drain_and_fold();
    }
    if (valid) {
      const uint32_t n = end - beg;
      const float inv = n ? 1.0f / (float)n : 0.0f;
      float* zrow = a.z + ((size_t)pix * a.mstride + a.j0) * 2 + (fb ? HV : 0);
#pragma unroll
      for (int i = 0; i < HV; i++) zrow[i] = mypart[i * RT_THREADS] * inv;
    }
    }
  }
}

template <int M>
static cudaError_t launch_routed_t(const SketchArgs& a, cudaStream_t s, int num_sms) {
  auto fn = sketch_routed_kernel<M>;
  const size_t smem = sketch_routed_smem(a.T, M);
  static SmemAttrOnce attr;
  cudaError_t e = smem_attr_once(attr, fn, 227 * 1024 - (RT_MAX_T + 16) / 16 * 16);  // minus the static cls
  if (e != cudaSuccess) return e;
  const long long tiles = (a.npix + 15) / 16;
  const long long need = (tiles + (RT_THREADS / 32) - 1) / (RT_THREADS / 32);
  long long grid = num_sms;  // one CTA per SM (shared memory)
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  fn<<<(unsigned)grid, RT_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

// One pass of M <= 32 frequencies, j0 = 0 only, T % 4 == 0 (the frame-B table
// is the quarter-period shift) and T <= RT_MAX_T (227 KB of shared memory).
cudaError_t launch_sketch_routed(int M, const SketchArgs& a, cudaStream_t s, int num_sms) {
  if (!routed_fits(a.T, a.j0)) return cudaErrorInvalidValue;
  switch (M) {
#define SRT3D_CASE(MM) \
  case MM:             \
    return launch_routed_t<MM>(a, s, num_sms);
    SRT3D_CASE(1) SRT3D_CASE(2) SRT3D_CASE(3) SRT3D_CASE(4) SRT3D_CASE(5) SRT3D_CASE(6) SRT3D_CASE(7) SRT3D_CASE(8)
    SRT3D_CASE(9) SRT3D_CASE(10) SRT3D_CASE(11) SRT3D_CASE(12) SRT3D_CASE(13) SRT3D_CASE(14) SRT3D_CASE(15)
    SRT3D_CASE(16) SRT3D_CASE(17) SRT3D_CASE(18) SRT3D_CASE(19) SRT3D_CASE(20) SRT3D_CASE(21) SRT3D_CASE(22)
    SRT3D_CASE(23) SRT3D_CASE(24) SRT3D_CASE(25) SRT3D_CASE(26) SRT3D_CASE(27) SRT3D_CASE(28) SRT3D_CASE(29)
    SRT3D_CASE(30) SRT3D_CASE(31) SRT3D_CASE(32)
#undef SRT3D_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace srt3d
