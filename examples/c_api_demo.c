/*
 * Minimal C user of the boundary (include/srt3d.h): no Python, no PyTorch.
 * Reads a CSR frame from a binary file, sketches it on the GPU (Eq. (3)),
 * evaluates the sketched loss + gradient at given parameters (Eq. (6)/(8)),
 * and writes z, grad_t, grad_alpha, loss to a binary output file.
 *
 *   input : int64 npix, uint32 T, m, K, float sigma, uint64 nph,
 *           uint32 offsets[npix+1], uint16 bins[nph], float t[npix*K], alpha[npix*K]
 *   output: float z[npix*m*2], grad_t[npix*K], grad_alpha[npix*K], loss[npix]
 *
 * Build: gcc -std=c11 c_api_demo.c -I../include -I/usr/local/cuda/include -L../paper_2203_00952_b200 -lsrt3d
 *            -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,<dir of libsrt3d.so>
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "srt3d.h"

#define CHECK_CUDA(x)                                                          \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "CUDA error %s at line %d\n", cudaGetErrorString(e_), __LINE__); \
      return 2;                                                                \
    }                                                                          \
  } while (0)
#define CHECK_SRT3D(x)                                                         \
  do {                                                                         \
    int r_ = (x);                                                              \
    if (r_ != SRT3D_OK) {                                                      \
      fprintf(stderr, "srt3d error %d: %s\n", r_, srt3d_last_error());         \
      return 3;                                                                \
    }                                                                          \
  } while (0)

static void* dev_copy(const void* h, size_t bytes) {
  void* d = NULL;
  if (cudaMalloc(&d, bytes ? bytes : 1) != cudaSuccess) return NULL;
  if (bytes && cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return NULL;
  return d;
}

int main(int argc, char** argv) {
  if (argc != 3) {
    fprintf(stderr, "usage: %s input.bin output.bin\n", argv[0]);
    return 1;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 1;
  int64_t npix;
  uint32_t T, m, K;
  float sigma;
  uint64_t nph;
  if (fread(&npix, 8, 1, f) != 1 || fread(&T, 4, 1, f) != 1 || fread(&m, 4, 1, f) != 1 || fread(&K, 4, 1, f) != 1 ||
      fread(&sigma, 4, 1, f) != 1 || fread(&nph, 8, 1, f) != 1)
    return 1;
  uint32_t* offsets = malloc(sizeof(uint32_t) * (npix + 1));
  uint16_t* bins = malloc(sizeof(uint16_t) * (nph ? nph : 1));
  float* t = malloc(sizeof(float) * npix * K);
  float* alpha = malloc(sizeof(float) * npix * K);
  if (fread(offsets, 4, npix + 1, f) != (size_t)(npix + 1) || fread(bins, 2, nph, f) != nph ||
      fread(t, 4, npix * K, f) != (size_t)(npix * K) || fread(alpha, 4, npix * K, f) != (size_t)(npix * K))
    return 1;
  fclose(f);

  uint16_t* d_bins = dev_copy(bins, 2 * nph);
  uint32_t* d_offsets = dev_copy(offsets, 4 * (npix + 1));
  float* d_t = dev_copy(t, 4 * npix * K);
  float* d_alpha = dev_copy(alpha, 4 * npix * K);
  float *d_z, *d_gt, *d_ga, *d_loss;
  CHECK_CUDA(cudaMalloc((void**)&d_z, sizeof(float) * npix * m * 2));
  CHECK_CUDA(cudaMalloc((void**)&d_gt, sizeof(float) * npix * K));
  CHECK_CUDA(cudaMalloc((void**)&d_ga, sizeof(float) * npix * K));
  CHECK_CUDA(cudaMalloc((void**)&d_loss, sizeof(float) * npix));
  if (!d_bins || !d_offsets || !d_t || !d_alpha) return 2;

  cudaStream_t s;
  CHECK_CUDA(cudaStreamCreate(&s));
  /* the north-star call: no photon-count hint, the regime is picked on the device */
  CHECK_SRT3D(srt3d_sketch(d_bins, d_offsets, npix, T, m, d_z, s));
  CHECK_SRT3D(srt3d_sketch_grad(d_z, d_t, d_alpha, npix, K, sigma, T, m, d_gt, d_ga, d_loss, s));
  /* an invalid call fails on the host, side-effect free, with a message */
  if (srt3d_sketch(d_bins, d_offsets, npix, T, T, d_z, s) != SRT3D_EINVAL) return 4;
  CHECK_CUDA(cudaStreamSynchronize(s));

  float* z = malloc(sizeof(float) * npix * m * 2);
  float* gt = malloc(sizeof(float) * npix * K);
  float* ga = malloc(sizeof(float) * npix * K);
  float* loss = malloc(sizeof(float) * npix);
  CHECK_CUDA(cudaMemcpy(z, d_z, sizeof(float) * npix * m * 2, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(gt, d_gt, sizeof(float) * npix * K, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(ga, d_ga, sizeof(float) * npix * K, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(loss, d_loss, sizeof(float) * npix, cudaMemcpyDeviceToHost));
  FILE* o = fopen(argv[2], "wb");
  if (!o) return 1;
  fwrite(z, 4, npix * m * 2, o);
  fwrite(gt, 4, npix * K, o);
  fwrite(ga, 4, npix * K, o);
  fwrite(loss, 4, npix, o);
  fclose(o);
  printf("srt3d %d: sketched %llu photons in %lld pixels\n", srt3d_version(), (unsigned long long)nph,
         (long long)npix);
  return 0;
}
