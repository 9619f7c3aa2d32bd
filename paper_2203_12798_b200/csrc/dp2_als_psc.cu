// Persistent ALS loop instances for R = 9..12 (see dp2_als_persist.cuh).
#include "dp2_als_persist.cuh"

namespace dp2 {
cudaError_t launch_persist_c(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st) {
  switch (R) {
#define DP2_PS_CASE(N) \
  case N: return launch_persist_t<N>(p, b, sms, st);
    DP2_PS_CASE(9) DP2_PS_CASE(10) DP2_PS_CASE(11) DP2_PS_CASE(12)
#undef DP2_PS_CASE
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace dp2
