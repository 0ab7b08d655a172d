// Tuning harness (tools only) for the bin-count sketch kernel: CTA size and
// loads in flight, on C3-like (256x256 px, T=2500, m=20, n=1e4) and C4-shaped
// frames (64x64 px, T=4096, m=10, n photons per pixel), half of the photons of
// a pixel in a 17-bin cluster.
#define HS_NO_DISPATCH
#include "../paper_2203_00952_b200/csrc/sketch_hist.cu"
#include <cstdio>
#include <random>
#include <vector>
using namespace srt3d;
#define CK(x)                                                           \
  do {                                                                  \
    cudaError_t e = (x);                                                \
    if (e != cudaSuccess) {                                             \
      printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__);     \
      exit(1);                                                          \
    }                                                                   \
  } while (0)
template <int M, int NT, int UNR>
void run(const SketchArgs& a, int nsm, double photons, const char* tag) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  {
    cudaError_t ee = launch_hist_t<M, NT, UNR>(a, 0, nsm);
    CK(ee);
  }
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) {
    cudaError_t ee = launch_hist_t<M, NT, UNR>(a, 0, nsm);
    CK(ee);
  }
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  double gbs = (2.0 * photons) / (ms * 1e-3) / 1e9;
  printf("{\"frame\":\"%s\",\"threads\":%d,\"unroll\":%d,\"ms\":%.4f,\"photons_per_s\":%.3e,\"gbs\":%.1f,\"frac_hbm\":%.3f}\n",
         tag, NT, UNR, ms, photons / (ms * 1e-3), gbs, gbs / 6547.8);
}
int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  struct F { long long npix, n; uint32_t T; const char* tag; };
  for (F fr : {F{65536, 10000, 2500, "C3like"}, F{4096, 10000, 4096, "C4@1e4"}, F{4096, 100000, 4096, "C4@1e5"}}) {
    const long long npix = fr.npix, n = fr.n;
    const uint32_t T = fr.T;
    std::vector<uint16_t> bins((size_t)npix * n);
    std::mt19937_64 g(7);
    for (long long i = 0; i < npix; i++) {
      uint16_t c = (uint16_t)(g() % T);
      for (long long p = 0; p < n; p++) {
        uint64_t r = g();
        bins[i * n + p] = (r & 1) ? (uint16_t)((r >> 8) % T) : (uint16_t)((c + T + (int)((r >> 20) % 17) - 8) % T);
      }
    }
    std::vector<uint32_t> offs(npix + 1);
    for (long long i = 0; i <= npix; i++) offs[i] = (uint32_t)(i * n);
    uint16_t* db;
    uint32_t* dof;
    float* dz;
    CK(cudaMalloc(&db, bins.size() * 2));
    CK(cudaMalloc(&dof, offs.size() * 4));
    CK(cudaMalloc(&dz, npix * 32 * 8));
    CK(cudaMemcpy(db, bins.data(), bins.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dof, offs.data(), offs.size() * 4, cudaMemcpyHostToDevice));
    double ph = (double)npix * n;
    if (T == 2500) {
      SketchArgs a{db, dof, npix, T, 0, 20u, dz};
      run<20, 512, 8>(a, nsm, ph, fr.tag);
      run<20, 256, 8>(a, nsm, ph, fr.tag);
      run<20, 128, 8>(a, nsm, ph, fr.tag);
      run<20, 128, 4>(a, nsm, ph, fr.tag);
      run<20, 64, 8>(a, nsm, ph, fr.tag);
    } else {
      SketchArgs a{db, dof, npix, T, 0, 10u, dz};
      run<10, 512, 8>(a, nsm, ph, fr.tag);
      run<10, 256, 8>(a, nsm, ph, fr.tag);
      run<10, 128, 8>(a, nsm, ph, fr.tag);
      run<10, 1024, 4>(a, nsm, ph, fr.tag);
    }
    cudaFree(db);
    cudaFree(dof);
    cudaFree(dz);
  }
  return 0;
}
