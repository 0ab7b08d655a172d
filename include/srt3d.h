/*
 * srt3d.h — C ABI of libsrt3d.so, the B200 (sm_100a) hot path of sketched
 * RT3D (SRT3D, arxiv 2203.00952).
 *
 * Citations: "PAPER.md:n" = line n of the paper text, "SPEC.md:n" = line n
 * of the CPU-program specification written from it; readings A1..A21 of
 * ambiguous or silent passages are listed in DESIGN.md §3.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA
 *    tensors).  The caller owns every buffer (workspace included, e.g. the
 *    bucketing scratch); the library allocates no device memory (except the
 *    measurement utility srt3d_debug_ffma_peak) and keeps no pointer after the
 *    call returns.
 *  - Calls are asynchronous and stream-ordered: work is enqueued on `stream`
 *    (a cudaStream_t; NULL = the legacy default stream) and the function
 *    returns without waiting for the device or reading device memory.
 *    Outputs are valid once the stream has synchronised.  Every compute entry
 *    point is legal inside CUDA-graph capture (srt3d_debug_ffma_peak, a
 *    synchronous measurement utility, is the one exception).
 *  - Reentrant: no global mutable state except the thread-local error string
 *    and per-device launch caches (atomics), so any number of host threads
 *    may call concurrently, on any streams and devices.
 *  - Layouts are row-major.  A sketch / expected sketch is complex64
 *    interleaved (re, im): float z[npix][m][2] (= torch.complex64 (npix, m)).
 *    Parameters are float t[npix][K], float alpha[npix][K].
 *  - Frequencies are the background-blind scheme omega_j = 2*pi*j/T,
 *    j = 1..m (reading A3).  t is in bins, omega in rad/bin.
 *  - Return value: SRT3D_OK (0) or a negative error code.  A failing call
 *    validates everything on the host BEFORE launching, so it writes nothing.
 *    srt3d_last_error() returns a thread-local message for the last failure.
 *  - npix == 0 is valid and a no-op.
 *  - Data preconditions that are NOT checked on the hot path (use
 *    srt3d_check_csr): 0 <= bins[p] < T, offsets non-decreasing,
 *    offsets[npix] - offsets[0] < 2^32.  Violations give unspecified values
 *    but never reads outside bins[offsets[0] .. offsets[npix]).
 *  - Inputs and outputs must not alias, except where an entry point says so
 *    (srt3d_descent_update / srt3d_sketch_grad_step / srt3d_fit_pixelwise
 *    update t and alpha in place; srt3d_sketch_merge may write over z_a or
 *    z_b; srt3d_sketch_accumulate updates (z, n) in place).
 */
#ifndef SRT3D_H_
#define SRT3D_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRT3D_OK 0
#define SRT3D_EINVAL (-1)       /* bad scalar argument (T, m, K, sigma, npix, eta) */
#define SRT3D_ENULL (-2)        /* required pointer is NULL */
#define SRT3D_EUNSUPPORTED (-3) /* m > SRT3D_MAX_M or K > SRT3D_MAX_K */
#define SRT3D_ECUDA (-4)        /* CUDA launch / runtime error (see srt3d_last_error) */
#define SRT3D_EALIGN (-5)       /* pointer not aligned to its element type */

#define SRT3D_MAX_T 65536u /* bins are uint16 */
#define SRT3D_MAX_M 64u
#define SRT3D_MAX_K 8u

/* Library version: major*10000 + minor*100 + patch. */
int srt3d_version(void);

/* Thread-local message describing the last non-zero return on this thread. */
const char* srt3d_last_error(void);

/*
 * srt3d_sketch — Eq. (3), the empirical characteristic
 * function of each pixel's photon time stamps:
 *     z[i][j-1] = (1/n_i) * sum_{p in pixel i} exp(i * 2*pi * j * x_p / T),
 *     j = 1..m,  n_i = offsets[i+1] - offsets[i].
 * An empty pixel (n_i = 0) gets z = 0 (reading A10).
 *   bins     uint16 photon bins, pixel-sorted CSR; pixel i owns
 *            bins[offsets[i] .. offsets[i+1]) (offsets[0] may be non-zero).
 *            Any 2-byte alignment.
 *   offsets  uint32 [npix + 1], 4-byte aligned.
 *   npix     number of pixels (>= 0).
 *   T        number of time bins, 2 <= T <= 65536.
 *   m        sketch size, 1 <= m <= min(T - 1, SRT3D_MAX_M).
 *   z        float [npix][m][2] output, 8-byte aligned; fully overwritten.
 *   stream   cudaStream_t (NULL = legacy default stream).
 * Arithmetic: the phase index r = (j*x) mod T is exact (integer); phasors
 * are fp32, accumulated in fp32 in a fixed (deterministic) order.
 * Launch regime (DESIGN.md §5.1/§5.3; lanes per pixel or the bin-count path,
 * chosen from the mean photons per pixel): selected ON THE DEVICE from
 * offsets[0] and offsets[npix] — the host enqueues the candidate kernels of
 * each 32-frequency pass and all but one exit at entry.  No host read, no
 * synchronisation.  srt3d_sketch_ex with a photon-count hint enqueues only
 * the selected kernel.
 * Data preconditions (not checked; see the conventions above): a bin >= T
 * yields unspecified finite values for its pixel, never an out-of-bounds
 * access.
 * Errors: SRT3D_EINVAL (T, m, npix), SRT3D_ENULL (bins, offsets or z NULL
 *         while npix > 0), SRT3D_EUNSUPPORTED (m > SRT3D_MAX_M),
 *         SRT3D_EALIGN, SRT3D_ECUDA.
 */
int srt3d_sketch(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, uint32_t m,
                 float* z, void* stream);

/*
 * srt3d_sketch_ex — srt3d_sketch with a host-side photon-count hint and/or
 * the launch regime chosen explicitly (same result up to fp32 rounding
 * order; used by the pipeline, tests and tuning):
 *   total_photons_hint  offsets[npix] - offsets[0] if the caller knows it:
 *                   the regime is then chosen on the host and only its kernel
 *                   is enqueued; SRT3D_HINT_UNKNOWN (0) selects on the device
 *                   as srt3d_sketch does.  A wrong hint changes the launch
 *                   shape only, never the result.
 *   path            SRT3D_PATH_AUTO (0): TENSOR when T <= 8192 and the mean
 *                   photon count per pixel is below 3 T; else bin-count when
 *                   the mean is >= T and the histogram fits in shared memory;
 *                   else ROUTED for a first pass of >= 24 frequencies at
 *                   256..2047 photons per pixel where it applies; else direct
 *                   (AUTO never selects PAIRED: measured slower, DESIGN.md
 *                   §5.1);
 *                   SRT3D_PATH_DIRECT (1): per-photon recurrence,
 *                   lanes_per_pixel lanes per pixel (0: by the photon count);
 *                   SRT3D_PATH_BINCOUNT (2): per-pixel shared-memory
 *                   histogram h[x] then z_j = (1/n) sum_x h[x] e^{i 2 pi j x/T}
 *                   (the same sum as Eq. (3) regrouped by bin; T <= ~17000,
 *                   else SRT3D_EUNSUPPORTED);
 *                   SRT3D_PATH_PAIRED (3): the direct sum, four lanes per
 *                   pixel, each chunk of <= 256 photons staged in shared
 *                   memory partitioned by phase class, then class-uniform
 *                   rotated Chebyshev loops with one accumulator frame switch
 *                   per class (T <= 23800, else
 *                   SRT3D_EUNSUPPORTED).
 *                   SRT3D_PATH_ROUTED (4): the direct sum, a lane pair per
 *                   pixel, each lane's accumulators in one of two rotation
 *                   frames and every photon routed (shared memory) to a lane
 *                   whose frame keeps its Chebyshev recurrence accurate:
 *                   one FFMA2 + one FADD2 per (photon, j) (
 *                   T % 4 == 0 and T <= 12000, else SRT3D_EUNSUPPORTED;
 *                   passes after the first 32 frequencies run the direct
 *                   path).
 *                   SRT3D_PATH_TENSOR (5): the bin-count sum on the tensor
 *                   cores: each pixel's photons are counted into a 32 x Kb
 *                   shared-memory histogram (Kb = 2^q >= T / 32) whose counts
 *                   are fed as fp16 bit patterns, multiplied on tcgen05 by the
 *                   per-column phasors e^{i w_j X_col} (hi + lo fp16 split),
 *                   and the 32 row sums twiddled by e^{i w_j X_row} and added
 *                   (T <= 8192, else SRT3D_EUNSUPPORTED; any
 *                   photon count: pixels above 2040 photons run in rounds).
 *   lanes_per_pixel 0 (auto) or 4, 8, 16, 32 (direct path); 0 or 2 (routed);
 *                   0 (tensor).
 * Errors as srt3d_sketch, plus SRT3D_EINVAL for an unknown path or lane count.
 */
#define SRT3D_PATH_AUTO 0
#define SRT3D_PATH_DIRECT 1
#define SRT3D_PATH_BINCOUNT 2
#define SRT3D_PATH_PAIRED 3
#define SRT3D_PATH_ROUTED 4
#define SRT3D_PATH_TENSOR 5
#define SRT3D_BINCOUNT_MIN_PHOTONS_PER_BIN 1.0
#define SRT3D_HINT_UNKNOWN 0ull
int srt3d_sketch_ex(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, uint32_t m, float* z,
                    uint64_t total_photons_hint, int path, int lanes_per_pixel, void* stream);

/*
 * srt3d_sketch_plan — host-only query: the path (SRT3D_PATH_DIRECT,
 * SRT3D_PATH_BINCOUNT, SRT3D_PATH_ROUTED or SRT3D_PATH_TENSOR) and lanes per pixel srt3d_sketch
 * would use for the first 32-frequency pass of a frame of npix pixels and
 * total_photons photons.  Returns the path (> 0) or a negative error code;
 * *lanes_per_pixel (may be NULL) receives the lane count (0 for the
 * bin-count path, which uses one CTA per pixel, and for the tensor-core path,
 * a warp pair per pixel slot of a 4-pixel tile; 2 for the routed path).
 */
int srt3d_sketch_plan(int64_t npix, uint32_t T, uint32_t m, uint64_t total_photons, int* lanes_per_pixel);

/*
 * srt3d_expected_sketch — Eq. (4) at omega_j = 2*pi*j/T with
 * the Gaussian IRF hhat(w) = exp(-sigma^2 w^2 / 2) (BASELINE.json north_star):
 *     z[i][j-1] = sum_{k<K} alpha[i][k] * hhat(omega_j) * exp(i omega_j t[i][k]).
 * The background term alpha_0 * CF_uniform(omega_j) is exactly 0 at these
 * frequencies (reading A4) and is not evaluated.  t may be any
 * real value (Phi is T-periodic in t; reading A16).
 *   t, alpha float [npix][K] (4-byte aligned);  K in 1..SRT3D_MAX_K.
 *   sigma    IRF standard deviation in bins, finite and >= 0.
 *   z        float [npix][m][2] output (8-byte aligned).
 */
int srt3d_expected_sketch(const float* t, const float* alpha, int64_t npix, uint32_t K, float sigma, uint32_t T,
                          uint32_t m, float* z, void* stream);

/*
 * srt3d_sketch_grad — the per-pixel sketched data-fidelity term of Eq. (6) /
 * Eq. (8) with W = I, unweighted by
 * n (reading A1), and its analytic gradient:
 *     r_j  = z_j - Phi_j(theta),            Phi_j as in srt3d_expected_sketch
 *     loss = sum_{j=1..m} |r_j|^2
 *     grad_alpha[k] = -2 sum_j hhat_j Re( conj(r_j) exp(i omega_j t_k) )
 *     grad_t[k]     = +2 alpha_k sum_j omega_j hhat_j Im( conj(r_j) exp(i omega_j t_k) )
 * (d/dalpha_0 = 0 because the background term vanishes at omega_j.)
 *   z        float [npix][m][2] (8-byte aligned), e.g. the srt3d_sketch output.
 *   t, alpha float [npix][K].
 *   grad_t, grad_alpha  float [npix][K] outputs.
 *   loss     float [npix] output, or NULL to skip it (reading A2: per pixel).
 */
int srt3d_sketch_grad(const float* z, const float* t, const float* alpha, int64_t npix, uint32_t K, float sigma,
                      uint32_t T, uint32_t m, float* grad_t, float* grad_alpha, float* loss, void* stream);

/*
 * srt3d_descent_update — the harness update step of the pixelwise data step
 * (reading A13; not an equation of the paper): in place, for every (i, k),
 *     t     -= clamp(eta * grad_t / (2 max(alpha,0.05)^2 sum_j omega_j^2 hhat_j^2), +-T/(4m)),
 *              then t is wrapped into [0, T)
 *     alpha  = clamp(alpha - eta * grad_alpha / (2 sum_j hhat_j^2), 0, 1)
 * using alpha's value before the update in both lines.
 *   eta finite and > 0.
 */
int srt3d_descent_update(float* t, float* alpha, const float* grad_t, const float* grad_alpha, int64_t npix,
                         uint32_t K, float sigma, uint32_t T, uint32_t m, float eta, void* stream);

/*
 * srt3d_sketch_grad_step — srt3d_sketch_grad followed by
 * srt3d_descent_update in ONE kernel (same arithmetic, grad_t / grad_alpha
 * never leave registers).  loss may be NULL.  t and alpha are updated in
 * place; each pixel's reads of t/alpha precede its writes.  For m % 16 == 0
 * (TMA z staging) the kernel is launched as a programmatic dependent of the
 * previous work on the stream: its CTAs may be scheduled during that work's
 * tail but read nothing before it has completed (griddepcontrol.wait), so
 * stream order is unchanged; the environment variable SRT3D_PDL=0 (read once
 * per process) launches it as an ordinary kernel.
 */
int srt3d_sketch_grad_step(const float* z, float* t, float* alpha, int64_t npix, uint32_t K, float sigma, uint32_t T,
                           uint32_t m, float eta, float* loss, void* stream);

/*
 * srt3d_fit_pixelwise — `iters` fused data steps in ONE launch (SURVEY §8(f)
 * NEXT-2, the pixelwise sketched fit of Eq. (6), with no
 * spatial coupling between iterations): z is staged once, t/alpha stay in
 * registers, and every iteration is exactly the srt3d_sketch_grad_step
 * arithmetic (the result equals `iters` srt3d_sketch_grad_step calls).
 * t and alpha are updated in place.  loss (optional, float [npix]) receives
 * the loss at the returned parameters.  iters <= 2^24.
 */
int srt3d_fit_pixelwise(const float* z, float* t, float* alpha, int64_t npix, uint32_t K, float sigma, uint32_t T,
                        uint32_t m, float eta, uint32_t iters, float* loss, void* stream);

/*
 * NEXT-3 — pixelwise initialisation of the sketched fit.  The
 * paper gives no initializer for Eq. (6); these follow the
 * matched-filter / phase readings A18-A20 of DESIGN.md.
 *
 * srt3d_backproject — g[i][n] = Re sum_{l=1..m} z_l hhat(omega_l) e^{-i omega_l t_n},
 * t_n = n*T/N, n = 0..N-1 (a circular grid), hhat Gaussian with sigma.
 *   z  float [npix][m][2] (8-byte aligned); g float [npix][N] output.
 *   1 <= N <= 8192.  Errors as srt3d_expected_sketch; N out of range: EINVAL.
 *   N % 32 == 0, N <= 512, m <= 32: computed on the tensor cores (tcgen05
 *   TF32 with a hi/lo split: fp32-level accuracy; the
 *   environment variable SRT3D_INIT_CUDA_CORES=1, read once per process,
 *   forces the CUDA-core kernel); other shapes on the CUDA cores.
 */
int srt3d_backproject(const float* z, int64_t npix, float sigma, uint32_t T, uint32_t m, uint32_t N, float* g,
                      void* stream);

/*
 * srt3d_init_depths — up to K initial depths per pixel from g (reading A19):
 * candidates are grid points with g_n > 0, g_n > g_{n-1}, g_n >= g_{n+1}
 * (circular); K times the largest (ties: smallest n) whose circular distance
 * d (grid steps) to every earlier pick has d*T >= min_sep*N.  Outputs, sorted
 * by depth: t [npix][K] = n*T/N, g_at [npix][K], alpha [npix][K] =
 * clamp(g_at / sum_l hhat_l^2, 0, 1), count [npix] (int32) = picks made.
 * Unfilled slots (reading A14): t = (t_first + T/2) mod T, g_at = alpha = 0.
 *   3 <= N <= 4096, 1 <= K <= SRT3D_MAX_K, min_sep in bins.  g as
 *   srt3d_backproject (tensor cores for N % 32 == 0, N <= 512, m <= 32).
 */
int srt3d_init_depths(const float* z, int64_t npix, float sigma, uint32_t T, uint32_t m, uint32_t N, uint32_t K,
                      uint32_t min_sep, float* t, float* g_at, float* alpha, int32_t* count, void* stream);

/*
 * srt3d_init_k1 — K = 1 closed form (reading A20):
 * t[i] = (T / 2 pi) arg(z_1) mapped into [0, T) (hhat_1 > 0 leaves the phase
 * unchanged); alpha[i] = clamp(sum_l hhat_l Re(conj(e^{i omega_l t}) z_l) /
 * sum_l hhat_l^2, 0, 1), the least-squares intensity at t.
 * |z_1| <= 1e-12: t = alpha = 0.   t, alpha float [npix] outputs.
 */
int srt3d_init_k1(const float* z, int64_t npix, float sigma, uint32_t T, uint32_t m, float* t, float* alpha,
                  void* stream);

/*
 * NEXT-4 — streaming acquisition: the sketch "can be updated in
 * an online fashion with each incoming photon".
 *
 * srt3d_sketch_merge — per pixel z_out = (n_a z_a + n_b z_b) / (n_a + n_b),
 * n_out = n_a + n_b (n = 0 -> z = 0): folds the sketch of a
 * new photon batch (n_b = its counts) into a running sketch.
 *   z_a, z_b, z_out float [npix][m][2] (8-byte aligned); n_a, n_b, n_out
 *   uint32 [npix].  z_out may alias z_a (or z_b) and n_out may alias n_a (or
 *   n_b): in-place accumulation.  Precondition: n_a + n_b < 2^32.
 */
int srt3d_sketch_merge(const float* za, const uint32_t* na, const float* zb, const uint32_t* nb, int64_t npix,
                       uint32_t m, float* z_out, uint32_t* n_out, void* stream);

/*
 * srt3d_sketch_accumulate — srt3d_sketch_merge in place into a running
 * (z, n) with the batch counts taken from the batch's CSR offsets,
 * n_b[i] = offsets_b[i+1] - offsets_b[i] (the offsets srt3d_sketch consumed to
 * produce z_b): the online update of PAPER.md:65 for one batch.
 */
int srt3d_sketch_accumulate(float* z, uint32_t* n, const float* zb, const uint32_t* offsets_b, int64_t npix,
                            uint32_t m, void* stream);

/*
 * srt3d_bucket_events — an unsorted stream of photon events (pixel index,
 * bin) into the pixel-sorted CSR frame srt3d_sketch consumes (reading A21),
 * by a two-level counting sort with coalesced writes:
 * offsets[i] = number of events with pixel < i, offsets[npix] = kept events,
 * and each pixel's bins contiguous in bins_out.  For npix <= 512 * 8192 the
 * sort is STABLE (each pixel's bins keep their stream order): the output is
 * deterministic, bit-identical run to run and to a stable counting sort;
 * larger frames use a one-level atomic scatter whose within-pixel order
 * follows atomic arrival (a permutation of the stable order; the sketch is
 * order-invariant up to fp32 rounding).  Events with pixel >= npix are
 * dropped and counted into *dropped (device uint32, may be NULL).
 *   pix uint32 [nevents], bins uint16 [nevents] (bins < T is the same
 *   precondition as for srt3d_sketch), nevents < 2^32; offsets uint32
 *   [npix+1] and bins_out uint16 [nevents] outputs; scratch uint32
 *   [srt3d_bucket_scratch_words(npix, nevents)] device workspace owned by the
 *   caller (about nevents + 512 * nevents / 32768 words).
 */
int srt3d_bucket_events(const uint32_t* pix, const uint16_t* bins, uint64_t nevents, int64_t npix,
                        uint32_t* offsets, uint16_t* bins_out, uint32_t* scratch, uint32_t* dropped, void* stream);
uint64_t srt3d_bucket_scratch_words(int64_t npix, uint64_t nevents);

/*
 * srt3d_check_csr — debug validator (not on the hot path).  Sets *bad (a
 * device int32 the caller zeroes first) to non-zero if some bins[p] >= T or
 * some offsets[i+1] < offsets[i].
 */
int srt3d_check_csr(const uint16_t* bins, const uint32_t* offsets, int64_t npix, uint32_t T, int32_t* bad,
                    void* stream);

/*
 * srt3d_debug_ffma_peak — measurement utility: the FP32
 * FMA throughput the current device sustains now, in TFLOP/s (2 flops per
 * FMA lane-op; 8 independent FFMA chains per thread on every SM, timed with
 * CUDA events on the legacy stream; synchronous; allocates 4 bytes).  The
 * bench reports the sketch's FP32 roofline against this and against the
 * unit-count peak.  Not part of the method.
 */
int srt3d_debug_ffma_peak(double* tflops);

/*
 * srt3d_debug_phase_index — test export of the exact integer phase index
 * used by srt3d_sketch: r[p][j-1] = (j * bins[p]) mod T, j = 1..m, computed
 * by the same device function the sketch kernel uses (PAPER.md:61 with
 * omega_j = 2 pi j / T).  r is uint32 [n][m].
 */
int srt3d_debug_phase_index(const uint16_t* bins, int64_t n, uint32_t T, uint32_t m, uint32_t* r, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SRT3D_H_ */
