// ba.cu — placeholder (kernel lands in the next milestone)
#include "common.cuh"
namespace rl {
int launch_ba(int32_t, int32_t, int64_t, const double *, const double *, const double *,
              const double *, const int32_t *, double, int32_t, double *, double *, double *, uint8_t *,
              unsigned long long *, cudaStream_t) {
  return set_error(RL_ERR_INVALID, "rl_ba_jac_f64: not implemented yet");
}
}  // namespace rl
