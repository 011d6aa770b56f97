// hjb_internal.cuh — host helpers shared by the C-ABI translation units
// (hjb_capi.cu defines them; hjb_shard.cu uses them).
#pragma once

#include <functional>
#include <vector>

#include "hjb_common.cuh"
#include "hjb_fast4d.cuh"

namespace hjb {

struct HostModel {
  DevModel dm;
  std::vector<double> tab;
  bool separable = true;
};

struct Scan {
  double max_speed_sum = 0.0;
  double max_alpha[kMaxDims] = {0};
};

// grid / model / bounds validated and uploaded; shape = fast-path id or -1
struct Prepared {
  DevGrid g;
  HostModel hm;
  int shape = -1;
};

int make_grid(const hjb_grid* gi, DevGrid& g);
int make_model(const hjb_model* mi, const hjb_dbounds* db, const DevGrid& g, HostModel& hm);
int validate_cfg(const hjb_solve_config* cfg);
int upload_model(hjb_context* ctx, HostModel& hm);
int run_scan(hjb_context* ctx, const DevGrid& g, const DevModel& m, Scan& out);
// Godunov + constant bounds preparation for the 4D fast path
int prepare(hjb_context* ctx, const hjb_grid* gi, const hjb_model* mi, const hjb_dbounds* db,
            Prepared& p);
void fill_tables(const Prepared& p, Fast4dArgs& f);
int scheme_of(const hjb_solve_config* cfg);
// Lax-Friedrichs fields of Fast4dArgs (f.lf = 0 for Godunov)
void fill_lf(const DevModel& m, int scheme, const double* galpha, Fast4dArgs& f);
// When the constraint c (reference layout, device) varies along axis 0 only
// (bit for bit), its per-plane values in ctx->cplane; else null.  Opt-in
// (HJB_CPLANE=1): measured no faster than the per-node field.
int constraint_planes(hjb_context* ctx, const DevGrid& g, const double* c, const double** out,
                      bool default_on = false);
// Grids whose solves run long enough to sit at the board's power cap (see
// hjb_capi.cu, constraint_planes): 4D first-order sweeps take 448 threads
// and, like the ENO3 stage (sustained 4441 vs 4575 us per 101^4 step,
// profiles/round2_ab_eno3.log), the per-plane constraint table there.
constexpr uint32_t kSustainedCells = 16u << 20;
void fill_lf(const DevModel& m, int scheme, const double* galpha, int& lf, LfParams& lp);
// Device iteration loop: WHILE-conditional CUDA graph (or HJB_LOOP=poll);
// `launch(stream, handle, use_handle)` enqueues one loop-mode sweep.
using SweepLauncher = std::function<cudaError_t(cudaStream_t, cudaGraphConditionalHandle, int)>;
int run_loop(hjb_context* ctx, const SweepLauncher& launch, int body);
int sm_count(int device);
// host per-node bounds -> context device buffer (constant bounds pass through)
int stage_dbounds(hjb_context* ctx, const hjb_dbounds* db, size_t n, DevBuf& buf,
                  hjb_dbounds& out);
int check_ctx(hjb_context* ctx);
inline int validate_config(const hjb_solve_config* cfg) { return validate_cfg(cfg); }

}  // namespace hjb
