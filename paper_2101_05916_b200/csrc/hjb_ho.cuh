// hjb_ho.cuh — high-order (ENO2/ENO3 + TVD-RK2/RK3) solver path.
// No reference implementation exists (reference SPEC.md:324, non-goal); the
// semantics are defined by the repo's own CPU restatement (oracle/hj_oracle.c).
#pragma once

#include "hjb_common.cuh"

namespace hjb {

int ho_solve(hjb_context* ctx, const DevGrid& g, const DevModel& m, const double* init,
             const double* c, const hjb_solve_config* cfg, double dt, const double* galpha,
             double* out, hjb_solve_result* res);

int ho_vi_step(hjb_context* ctx, const DevGrid& g, const DevModel& m, const double* v,
               const double* c, const hjb_solve_config* cfg, double dt, const double* galpha,
               double* out);

}  // namespace hjb
