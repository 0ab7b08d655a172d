// Internal declarations shared by the kernel translation units and the C ABI.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace srt3d {

constexpr int SK_THREADS = 256;                 // sketch CTA size
constexpr size_t SK_MAX_SMEM = 24576 * 8;       // phase-table bytes (T < 24576 uses the smem table)
#ifndef SK_SCHEME
#define SK_SCHEME 0                              // grouped direct path phasor scheme: 0 complex power, 1 rotated Chebyshev (selects)
#endif
constexpr uint32_t SO_MAX_T = 23800;             // class-sorted path: phase table + per-group photon buffers fit 227 KB
constexpr int SK_G4_CHEB = -4;                  // launch_sketch_pass regime: G = 4 with the rotated Chebyshev scheme
constexpr int PX_THREADS = 128;                 // pixel-kernel CTA size
#ifndef GRAD_THREADS
#define GRAD_THREADS 64                          // gradient-kernel CTA size (one warp = 32 pixels)
#endif
#ifndef GRAD_TMA_MIN_BLOCKS
#define GRAD_TMA_MIN_BLOCKS 10                   // TMA variant: 96 registers (12 measured slower in loop: tools/grad_probe.py)
#endif
#ifndef GRAD_PERSIST
#define GRAD_PERSIST 0  // 1: one wave of TMA-gradient CTAs, each warp looping over tiles (measured slower:
                        // C5 22.4 us cold, 16.4 in loop vs 18.0 / 13.55 — per-warp tiles in sequence expose the loads)
#endif
#ifndef GRAD_PDL_TRIGGER
#define GRAD_PDL_TRIGGER 0  // 1: each TMA-gradient CTA fires griddepcontrol.launch_dependents once its tile
                            // loads are issued, so the next step's CTAs are scheduled during this one's tail
#endif
#ifndef GRAD_MIN_BLOCKS
#define GRAD_MIN_BLOCKS 12                       // smem caps residency at 12 CTAs/SM: let ptxas use up to 80 regs
#endif
constexpr int MAX_M = 64;
constexpr int MAX_K = 8;

struct SketchArgs {
  const uint16_t* bins;
  const uint32_t* offsets;
  long long npix;
  uint32_t T;
  uint32_t j0;       // first frequency of this pass is j0 + 1
  uint32_t mstride;  // m of the output row
  float* z;
  // Device-side regime selection (srt3d_sketch without a photon-count hint):
  // rg_want != RG_NONE makes the kernel exit unless sketch_regime(offsets[npix] -
  // offsets[0], npix, T, M, rg_mode) == rg_want, so exactly one of the candidate
  // launches of a pass does the work and the host never reads device memory.
  uint32_t rg_mode;  // RGM_AUTO / RGM_DIRECT / RGM_HIST
  uint32_t rg_want;  // RG_NONE: unconditional launch
};

// ---- launch regimes of the sketch -------------------
// A function of the frame's photon count, evaluated with exact integer
// comparisons so the host (with a hint) and the device (from offsets) agree:
// mean >= X  <=>  total >= X * npix.
enum : uint32_t { RG_NONE = 0, RG_G4, RG_G8, RG_G16, RG_G32, RG_G4C, RG_RT, RG_TC, RG_H128, RG_H256, RG_H512, RG_COUNT };
// class-routed Chebyshev kernel (sketch_routed.cu): first pass only, T % 4 == 0, T <= RT_MAX_T
constexpr uint32_t RT_MAX_T = 12000;  // 1.25 T phasor entries + T class bytes + [32][512] fp32 partials + spills <= 227 KB
__host__ __device__ inline bool routed_fits(uint32_t T, uint32_t j0) { return j0 == 0 && T % 4 == 0 && T <= RT_MAX_T; }
// tensor-core sketch (sketch_tc.cu): a pixel's bins fill a 32 x Kb fp16 block, Kb = 2^q <= 256
constexpr uint32_t TC_MAX_T = 8192;
__host__ __device__ inline bool tc_fits(uint32_t T) { return T >= 1 && T <= TC_MAX_T; }
constexpr unsigned long long TC_MAX_MEAN_PER_T = 3;  // AUTO: tensor-core path below 3 T photons per pixel (measured)
enum : uint32_t { RGM_AUTO = 0, RGM_DIRECT = 1, RGM_HIST = 2 };
constexpr uint32_t SK_TABLE_MAX_T = 24575;  // (T + 1) float2 entries fit SK_MAX_SMEM
// mode: RGM_AUTO (bin-count allowed: the host passes it only when the
// histogram fits in shared memory), RGM_DIRECT, RGM_HIST (bin-count forced).
__host__ __device__ inline uint32_t sketch_regime(unsigned long long total, long long npix, uint32_t T, int M,
                                                  uint32_t mode, uint32_t j0) {
  const unsigned long long np = npix > 0 ? (unsigned long long)npix : 1ull;
  // tensor-core sketch (§5.7): measured fastest at every BASELINE config with T <= 8192 and a mean
  // below 3 T photons per pixel (above it the bin-count path's HBM-bound histogram wins)
  if (mode == RGM_AUTO && tc_fits(T) && total < TC_MAX_MEAN_PER_T * T * np) return RG_TC;
  const bool hist = mode == RGM_HIST || (mode == RGM_AUTO && total >= (unsigned long long)T * np);
  if (hist) {
    if (total < 30000ull * np) return RG_H128;  // CTA size by photons per pixel (tools/hist_tune.cu)
    if (total < 80000ull * np) return RG_H256;
    return RG_H512;
  }
  if (T > SK_TABLE_MAX_T) return RG_G32;  // no shared phase table: one configuration
  if (total >= 4096ull * np) return RG_G32;
  if (total >= 2048ull * np) return RG_G16;
  // long passes: the class-routed Chebyshev kernel where it fits, else G = 4 rotated Chebyshev
  if (total >= 256ull * np) return M >= 24 ? (routed_fits(T, j0) ? RG_RT : RG_G4C) : RG_G8;
  return RG_G4;
}

// Device side: true if this launch is a candidate that was not selected.
__device__ __forceinline__ bool sketch_regime_skip(const SketchArgs& a, int M) {
  if (a.rg_want == RG_NONE) return false;
  const uint32_t tot = a.offsets[a.npix] - a.offsets[0];  // < 2^32 (precondition)
  return sketch_regime(tot, a.npix, a.T, M, a.rg_mode, a.j0) != a.rg_want;
}

// Per-call frequency constants, computed on the host in fp64 and rounded:
// hh[j-1] = hhat(omega_j) = exp(-sigma^2 omega_j^2 / 2), wh[j-1] = omega_j * hhat(omega_j).
struct FreqConsts {
  float hh[MAX_M];
  float wh[MAX_M];
};

struct PixArgs {
  const float* z;     // [npix][m][2] (grad) or output (expected sketch)
  float* zout;
  const float* t_in;
  const float* a_in;
  float* t_out;       // update modes
  float* a_out;
  float* grad_t;
  float* grad_a;
  float* loss;
  long long npix;
  uint32_t T;
  uint32_t m;
  double invT;
  float eta;
  float upd_t_scale;  // 1 / (2 * sum_j omega_j^2 hhat_j^2)
  float upd_a_scale;  // 1 / (2 * sum_j hhat_j^2)
  float max_step;     // T / (4 m)
  float Tf;
  float invTf;        // 1 / T (fp32)
  FreqConsts c;
};

enum PixMode { PX_EXPECTED = 0, PX_GRAD = 1, PX_GRAD_STEP = 2, PX_UPDATE = 3, PX_GRAD_STEP_NL = 4, PX_GRAD_NL = 5 };  // NL: no loss output

// Per-device host-side launch caches.  cudaFuncSetAttribute acts on the
// current device only, and the resident-CTA count is a per-device property, so
// both are keyed by cudaGetDevice(); entries are lock-free atomics (a race only
// repeats idempotent work), so concurrent callers on any devices are safe.
constexpr int MAX_DEVICES = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= MAX_DEVICES) d = 0;
  return d;
}

// "Raise this kernel's dynamic shared-memory limit to `bytes`" once per device.
struct SmemAttrOnce {
  std::atomic<int> done[MAX_DEVICES];
};
template <typename F>
inline cudaError_t smem_attr_once(SmemAttrOnce& o, F fn, int bytes) {
  const int d = current_device();
  if (o.done[d].load(std::memory_order_acquire)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  o.done[d].store(1, std::memory_order_release);
  return cudaSuccess;
}

// Resident CTAs per SM of one kernel for the last dynamic shared-memory size
// asked for on each device (the occupancy query costs several microseconds per
// launch otherwise).  One 64-bit word per device: (smem + 1) << 16 | per_sm,
// so a reader never sees a count paired with another size.
struct OccCache {
  std::atomic<unsigned long long> v[MAX_DEVICES];
};
template <typename F>
inline cudaError_t occupancy_cached(OccCache& c, F fn, int threads, size_t smem, int* per_sm) {
  const int d = current_device();
  const unsigned long long cur = c.v[d].load(std::memory_order_relaxed);
  if (cur != 0 && (cur >> 16) == (unsigned long long)smem + 1) {
    *per_sm = (int)(cur & 0xffffu);
    return cudaSuccess;
  }
  int v = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (v < 1) v = 1;
  c.v[d].store((((unsigned long long)smem + 1) << 16) | (unsigned long long)(v & 0xffff), std::memory_order_relaxed);
  *per_sm = v;
  return cudaSuccess;
}

// SM count of the current device (cached per device).
inline int num_sms_device() {
  static std::atomic<int> cache[MAX_DEVICES];
  const int d = current_device();
  int n = cache[d].load(std::memory_order_relaxed);
  if (n > 0) return n;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n <= 0) n = 148;
  cache[d].store(n, std::memory_order_relaxed);
  return n;
}

cudaError_t launch_sketch_pass(int M, int G, const SketchArgs& a, cudaStream_t s, int num_sms);
cudaError_t measure_ffma_peak(double* tflops, int num_sms);
cudaError_t launch_sketch_hist(int M, const SketchArgs& a, int threads, cudaStream_t s, int num_sms);
size_t sketch_hist_smem(uint32_t T, int M);
cudaError_t launch_sketch_pair(int M, const SketchArgs& a, cudaStream_t s, int num_sms);
// class-routed Chebyshev sketch (sketch_routed.cu): a lane pair per pixel, j0 = 0, T % 4 == 0, T <= RT_MAX_T
cudaError_t launch_sketch_routed(int M, const SketchArgs& a, cudaStream_t s, int num_sms);
size_t sketch_routed_smem(uint32_t T, int M);
size_t sketch_pair_smem(uint32_t T);
// tensor-core sketch (sketch_tc.cu): T <= TC_MAX_T, one pass of M <= 32 frequencies
cudaError_t launch_sketch_tc(int M, const SketchArgs& a, cudaStream_t s, int num_sms);
size_t sketch_tc_smem(uint32_t T, int MP);
cudaError_t launch_phase_index(const uint16_t* bins, long long n, uint32_t T, uint32_t m, uint32_t* r,
                               cudaStream_t s, int num_sms);
cudaError_t launch_check_csr(const uint16_t* bins, const uint32_t* offsets, long long npix, uint32_t T,
                             int32_t* bad, cudaStream_t s, int num_sms);
cudaError_t launch_pixel(PixMode mode, int K, const PixArgs& a, cudaStream_t s);
// NEXT-3 initialisation kernels (init.cu).
struct BpArgs {
  const float* z;   // [npix][m][2]
  float* g;         // backprojection output [npix][N] (or null)
  float* t_out;     // picks [npix][K] (init_depths) or [npix] (init_k1)
  float* g_out;
  float* a_out;
  int32_t* count;
  long long npix;
  uint32_t T, m, N, K, min_sep;
  float inv_sh2;    // 1 / sum_l hhat_l^2
  float hh[MAX_M];  // hhat_l
  int list_cap;     // tensor-core init_depths: candidate-list entries per thread (set by its launcher)
};
cudaError_t launch_backproject(const BpArgs& a, bool pick, cudaStream_t s, int num_sms);
// tensor-core backprojection (init_tc.cu): N % 32 == 0, 32 <= N <= 512, m <= 32
bool backproject_tc_supported(uint32_t N, uint32_t m);
cudaError_t launch_backproject_tc(const BpArgs& a, bool pick, cudaStream_t s, int num_sms);
cudaError_t launch_init_k1(const BpArgs& a, cudaStream_t s);
size_t backproject_smem(uint32_t N, bool pick);
// NEXT-4 streaming acquisition (stream.cu).
cudaError_t launch_merge(const float* za, const uint32_t* na, const float* zb, const uint32_t* nb,
                         const uint32_t* offs_b, long long npix, uint32_t m, float* zo, uint32_t* no, cudaStream_t s,
                         int num_sms);
size_t bucket_scratch_words(long long npix, unsigned long long nev);
cudaError_t launch_bucket(const uint32_t* pix, const uint16_t* bins, unsigned long long nev, long long npix,
                          uint32_t* offsets, uint16_t* bins_out, uint32_t* scratch, uint32_t* dropped_out,
                          cudaStream_t s, int num_sms);
cudaError_t launch_fit(int K, const PixArgs& a, int iters, cudaStream_t s);

}  // namespace srt3d
