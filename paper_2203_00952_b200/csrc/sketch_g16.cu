// K1 instantiations for G = 16 lanes per pixel (split for parallel builds).
#include "sketch_impl.cuh"

namespace srt3d {
cudaError_t launch_sketch_g16(int M, bool tab, const SketchArgs& a, cudaStream_t s, int num_sms) {
  return dispatch_m<16, true, SK_SCHEME>(M, a, s, num_sms);
}
}  // namespace srt3d
