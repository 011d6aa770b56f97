// hjb_kernels.cuh — launch interface of the sm_100a kernels (hjb_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "hjb_device.cuh"

namespace hjb {

enum Scheme { kGodunov = 0, kLfPerNode = 1, kLfGlobal = 2 };

// Arguments of one VI sweep (solver.cpp:106-190 over the whole grid).
struct StepArgs {
  DevGrid g;
  DevModel m;
  const double* c;   // constraint
  // target set l (reach-avoid extension, no reference counterpart): the
  // update is max(c, min(l, stepped)); null = the reference update
  const double* target;
  double* buf0;      // loop mode: front/back double buffer, parity = st->iter
  double* buf1;
  const double* src; // single-step mode
  double* dst;
  LoopState* st;
  double dt;
  double galpha[kMaxDims];
  int scheme;
  int loop;          // 1: read parity/done from st and run the epilogue
  cudaGraphConditionalHandle handle;
  int use_handle;
  // high-order stages (k_ho_stage): buffers and roles
  double* stage1;
  double* stage2;
  int src_sel;      // 0: V_n (parity / src), 1: stage1, 2: stage2
  int dst_sel;      // 0: V_{n+1} (parity / dst), 1: stage1, 2: stage2
  int kind;         // 0 first stage, 1 RK2 final, 2 RK3 second, 3 RK3 final
  int final_stage;  // run the max|dV| reduction / loop epilogue
  int order;        // ENO order 1..3
};

// Whole solve() loop of a small 2D grid in one cluster launch (<= 16 CTAs,
// V in distributed shared memory).  s.src = init, s.dst = out (device),
// s.st = loop state initialised by launch_loop_init.  small2d_smem returns
// the per-CTA shared memory (0 when the grid is not 2D).
size_t small2d_smem(const DevGrid& g, uint32_t* rows, uint32_t* ctas);
cudaError_t launch_small2d(const StepArgs& s, cudaStream_t stream);
// ENO/TVD-RK variant (s.order = ENO order, rk = TVD-RK order): all stages of
// the whole loop in one cluster launch; 0 smem when the grid is not 2D
size_t small2d_ho_smem(const DevGrid& g, uint32_t* rows, uint32_t* ctas);
cudaError_t launch_small2d_ho(const StepArgs& s, int rk, cudaStream_t stream);

// K6: one ENO/TVD-RK stage (generic rank; see hjb_kernels.cu).
cudaError_t launch_ho_stage(const StepArgs& a, cudaStream_t s);

// K1: alpha scan (solver.cpp:221-268).  out[0] = max_nodes sum_d alpha_d/dx_d,
// out[1+d] = max_nodes alpha_d.  out must be zeroed by the caller.
cudaError_t launch_scan(const DevGrid& g, const DevModel& m, double* out, cudaStream_t s);

// K2/K3: one Euler sweep with the VI clamp and the max|dV| reduction.
cudaError_t launch_step(const StepArgs& a, cudaStream_t s);

// Loop state initialisation (records the start timestamp on the device).
cudaError_t launch_loop_init(LoopState* st, long long max_iters, double dt, double tol,
                             double horizon, long long history_cap, double* history,
                             double* wall_history, cudaStream_t s);

// K4: multilinear resample (grid.cpp:84-135,215-231); optional seed clamp
// out = max(resampled - *slack, c) when c != nullptr (solver.cpp:404-411).
cudaError_t launch_resample(const DevGrid& src_g, const double* src, const DevGrid& dst_g,
                            double* dst, const double* slack, const double* c,
                            cudaStream_t s);

// max_adjacent_jump (grid.cpp:197-213) into *out (zeroed by the caller).
cudaError_t launch_max_adjacent_jump(const DevGrid& g, const double* f, double* out,
                                     cudaStream_t s);

// K5: signed_distance_band / field_max / field_min (levelset.cpp:54-95).
cudaError_t launch_band(const DevGrid& g, int dim, double lo, double hi, double* out,
                        cudaStream_t s);
cudaError_t launch_field_op(long long n, const double* a, const double* b, double* out,
                            int is_max, cudaStream_t s);

// fill n doubles with a value
cudaError_t launch_fill(double* out, uint32_t n, double value, cudaStream_t s);
// *flag |= 1 if any of f[0..n) differs bitwise from f[0] (flag zeroed by caller)
cudaError_t launch_not_constant(const double* f, uint32_t n, unsigned int* flag, cudaStream_t s);
cudaError_t launch_not_axis0(const double* f, uint32_t n, uint32_t s0, unsigned int* flag,
                             cudaStream_t s);

}  // namespace hjb
