// K1 instantiations for G = 32 lanes per pixel (split for parallel builds).
#include "sketch_impl.cuh"

namespace srt3d {
cudaError_t launch_sketch_g32(int M, bool tab, const SketchArgs& a, cudaStream_t s, int num_sms) {
  if (!tab) return dispatch_m<32, false, SK_SCHEME>(M, a, s, num_sms);
  return dispatch_m<32, true, SK_SCHEME>(M, a, s, num_sms);
}
}  // namespace srt3d
