// kernels_tc.cu — tcgen05/TMEM/TMA tensor-core convolutions (placeholder, being written).
#include "kernels.cuh"

namespace cp {
size_t tc_workspace_bytes(const Layer&) { return 0; }
int tc_fwd(Layer&, const float*, const float*, const float*, float*, uint8_t*, void*, cudaStream_t) {
  CP_FAIL(CP_ERR_UNSUPPORTED, "tcgen05 forward not built yet");
}
int tc_dgrad(Layer&, const float*, const float*, float*, void*, cudaStream_t) {
  CP_FAIL(CP_ERR_UNSUPPORTED, "tcgen05 dgrad not built yet");
}
int tc_wgrad(Layer&, const float*, const float*, float*, void*, cudaStream_t) {
  CP_FAIL(CP_ERR_UNSUPPORTED, "tcgen05 wgrad not built yet");
}
void tc_release(Layer&) {}
}  // namespace cp
