// Persistent ALS loop instances for R = 13..16 (see dp2_als_persist.cuh).
#include "dp2_als_persist.cuh"

namespace dp2 {
cudaError_t launch_persist_d(int R, const PsArgs& p, const AlsBufs& b, int sms, cudaStream_t st) {
  switch (R) {
#define DP2_PS_CASE(N) \
  case N: return launch_persist_t<N>(p, b, sms, st);
    DP2_PS_CASE(13) DP2_PS_CASE(14) DP2_PS_CASE(15) DP2_PS_CASE(16)
#undef DP2_PS_CASE
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace dp2
