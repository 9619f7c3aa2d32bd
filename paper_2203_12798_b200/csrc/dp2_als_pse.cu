// Persistent ALS loop instance for R = 20 (see dp2_als_persist.cuh).  The
// register Jacobi keeps one column per lane, so the loop itself covers R <= 32;
// above R = 16 only R = 20 and 24 are instantiated (each costs minutes of
// ptxas time at 255 registers); other ranks take the seven-kernel loop.
// Measured at c4 (K = 1000, J = 512, p = R): R = 20, 557 us per iteration
// against 1117 us for the seven-kernel loop.
#include "dp2_als_persist.cuh"

namespace dp2 {
cudaError_t launch_persist_e(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st) {
  return R == 20 ? launch_persist_t<20>(p, b, sms, st) : cudaErrorInvalidValue;
}
}  // namespace dp2
