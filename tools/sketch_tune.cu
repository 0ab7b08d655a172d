// Tuning harness (tools only): times sketch_kernel variants (lanes per pixel G,
// phasor scheme SCH: 0 complex power, 1 rotated Chebyshev) on a C5-shaped synthetic frame (uniform random bins,
// T=8192, m=32, 262144 px x 1000 photons) and on an m=10 / n=1e4 frame, and
// cross-checks every variant against the TP=0 result.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../paper_2203_00952_b200/csrc/sketch_impl.cuh"

using namespace srt3d;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int M, int G, int SCH>
float time_variant(const SketchArgs& a, int nsm, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  { cudaError_t ee = launch_sketch_t<M, G, true, SCH>(a, 0, nsm); CK(ee); }
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < reps; r++) { cudaError_t ee = launch_sketch_t<M, G, true, SCH>(a, 0, nsm); CK(ee); }
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

template <int M, int G, int SCH>
void run(const char* tag, SketchArgs a, int nsm, double photons, std::vector<float>& ref, float* z, size_t zn) {
  float ms = time_variant<M, G, SCH>(a, nsm, 5);
  std::vector<float> h(zn);
  CK(cudaMemcpy(h.data(), z, zn * 4, cudaMemcpyDeviceToHost));
  double d = 0;
  if (ref.empty()) ref = h; else for (size_t i = 0; i < zn; i++) d = fmax(d, fabs(h[i] - ref[i]));
  double tflops = 8.0 * M * photons / (ms * 1e-3) / 1e12;
  printf("{\"frame\":\"%s\",\"M\":%d,\"G\":%d,\"SCH\":%d,\"ms\":%.4f,\"tflops\":%.2f,\"frac_fp32_1965\":%.4f,\"maxdiff_vs_first\":%.2e}\n",
         tag, M, G, SCH, ms, tflops, tflops / 74.45, d);
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  for (int frame = 0; frame < 2; frame++) {
    const uint32_t T = frame == 0 ? 8192 : 4096;
    const long long npix = frame == 0 ? 262144 : 16384;
    const int n = frame == 0 ? 1000 : 10000;
    std::vector<uint16_t> bins((size_t)npix * n);
    uint64_t st = 12345;
    for (auto& b : bins) { st = st * 6364136223846793005ULL + 1442695040888963407ULL; b = (uint16_t)((st >> 33) % T); }
    std::vector<uint32_t> offs(npix + 1);
    for (long long i = 0; i <= npix; i++) offs[i] = (uint32_t)(i * n);
    uint16_t* db; uint32_t* dof; float* dz;
    CK(cudaMalloc(&db, bins.size() * 2)); CK(cudaMalloc(&dof, offs.size() * 4));
    const int m = frame == 0 ? 32 : 10;
    size_t zn = (size_t)npix * m * 2;
    CK(cudaMalloc(&dz, zn * 4));
    CK(cudaMemcpy(db, bins.data(), bins.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dof, offs.data(), offs.size() * 4, cudaMemcpyHostToDevice));
    SketchArgs a{db, dof, npix, T, 0, (uint32_t)m, dz};
    std::vector<float> ref;
    double ph = (double)npix * n;
    if (frame == 0) {
      run<32, 8, 0>("C5like", a, nsm, ph, ref, dz, zn);
      run<32, 4, 1>("C5like", a, nsm, ph, ref, dz, zn);
      run<32, 2, 1>("C5like", a, nsm, ph, ref, dz, zn);
      run<32, 1, 1>("C5like", a, nsm, ph, ref, dz, zn);
      run<32, 2, 0>("C5like", a, nsm, ph, ref, dz, zn);
      run<32, 4, 1>("C5like", a, nsm, ph, ref, dz, zn);
      run<32, 16, 1>("C5like", a, nsm, ph, ref, dz, zn);
      run<32, 8, 2>("C5like", a, nsm, ph, ref, dz, zn);
      run<32, 4, 2>("C5like", a, nsm, ph, ref, dz, zn);
    } else {
      run<10, 16, 0>("m10n1e4", a, nsm, ph, ref, dz, zn);
      run<10, 16, 1>("m10n1e4", a, nsm, ph, ref, dz, zn);
      run<10, 8, 1>("m10n1e4", a, nsm, ph, ref, dz, zn);
      run<10, 32, 1>("m10n1e4", a, nsm, ph, ref, dz, zn);
    }
    cudaFree(db); cudaFree(dof); cudaFree(dz);
  }
  return 0;
}
