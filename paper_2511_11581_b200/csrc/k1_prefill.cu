// K1 -- tcgen05/TMEM prefill Q-block kernel (§4.4).  (in progress)
#include "common.cuh"
#include "kernels.h"

namespace pattn {

bool prefill_supported(const Params&) { return false; }

PrefillLaunch plan_prefill(const Params&, int num_sms) {
  PrefillLaunch pl;
  pl.grid = num_sms;
  pl.smem = 0;
  return pl;
}

cudaError_t launch_prefill(const Params&, const PrefillLaunch&, const CUtensorMap&, const CUtensorMap&,
                           const CUtensorMap&, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace pattn
