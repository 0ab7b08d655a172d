// Internal declarations shared by the kernel translation units and the C ABI.
#pragma once
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
#define GRAD_TMA_MIN_BLOCKS 10                   // TMA variant: swizzled addressing needs a few more registers
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
};

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

// Host-side cache of the resident-CTA count of one kernel for the last
// dynamic shared-memory size asked for (the occupancy query costs several
// microseconds per launch otherwise).  Races are benign: a stale or torn
// value only changes a persistent grid's size, never a result.
struct OccCache {
  size_t smem = ~(size_t)0;
  int per_sm = 0;
};
template <typename F>
inline cudaError_t occupancy_cached(OccCache& c, F fn, int threads, size_t smem, int* per_sm) {
  if (c.smem == smem && c.per_sm > 0) {
    *per_sm = c.per_sm;
    return cudaSuccess;
  }
  int v = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (v < 1) v = 1;
  c.per_sm = v;
  c.smem = smem;
  *per_sm = v;
  return cudaSuccess;
}

cudaError_t launch_sketch_pass(int M, int G, const SketchArgs& a, cudaStream_t s, int num_sms);
cudaError_t measure_ffma_peak(double* tflops, int num_sms);
cudaError_t launch_sketch_hist(int M, const SketchArgs& a, double mean_photons, cudaStream_t s, int num_sms);
size_t sketch_hist_smem(uint32_t T, int M);
cudaError_t launch_sketch_pair(int M, const SketchArgs& a, cudaStream_t s, int num_sms);
size_t sketch_pair_smem(uint32_t T);
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
