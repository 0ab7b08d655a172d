// K1 instantiations for G = 4 lanes per pixel with the rotated Chebyshev
// scheme (per-photon rotation by selects): the fastest direct variant for
// m >= 24 at ~1e3 photons per pixel (C5: 1.56 vs 1.61 ms for the complex
// power at G = 8; tools/sketch_tune.cu).
#include "sketch_impl.cuh"

namespace srt3d {
cudaError_t launch_sketch_g4_cheb(int M, const SketchArgs& a, cudaStream_t s, int num_sms) {
  return dispatch_m<4, true, SCH_CHEB>(M, a, s, num_sms);
}
}  // namespace srt3d
