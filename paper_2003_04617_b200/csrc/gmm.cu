// gmm.cu — placeholder (kernel lands in a later milestone)
#include "common.cuh"
namespace rl {
size_t gmm_workspace_bytes(int32_t, int32_t, int64_t) { return 0; }
int launch_gmm(int32_t, int32_t, int64_t, int64_t, const double *, const double *, const double *,
               const double *, double, int32_t, double, double, int32_t, int32_t, double *,
               uint8_t *, unsigned long long *, void *, size_t, cudaStream_t) {
  return set_error(RL_ERR_INVALID, "rl_gmm_grad_f64: not implemented yet");
}
}  // namespace rl
