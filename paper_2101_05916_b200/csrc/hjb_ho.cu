// hjb_ho.cu — high-order solver path (see hjb_ho.cuh).
#include "hjb_ho.cuh"

namespace hjb {

int ho_solve(hjb_context*, const DevGrid&, const DevModel&, const double*, const double*,
             const hjb_solve_config*, double, const double*, double*, hjb_solve_result*) {
  return set_err(HJB_ERR_UNSUPPORTED, "solve: spatial/time order > 1 not available yet");
}

int ho_vi_step(hjb_context*, const DevGrid&, const DevModel&, const double*, const double*,
               const hjb_solve_config*, double, const double*, double*) {
  return set_err(HJB_ERR_UNSUPPORTED, "vi_step: spatial/time order > 1 not available yet");
}

}  // namespace hjb
