// hjb_device.cuh — device-side data structures shared by the sm_100a kernels.
//
// Everything here is plain data handed to kernels by value.  The arithmetic
// contract with the reference (hjsafe, proj/src/solver.cpp) is bitwise: the
// library is compiled with -fmad=false so every a*b+c stays a DMUL followed
// by a DADD, exactly like the reference compiled without FMA contraction.
#pragma once

#include <cstdint>

#include "../../include/hjb.h"

namespace hjb {

constexpr int kMaxDims = HJB_MAX_DIMS;
constexpr int kMaxState = HJB_MAX_STATE;
constexpr int kMaxInput = HJB_MAX_INPUT;

// Unsigned 32-bit division by a loop-invariant divisor (multiply-high and
// shift), valid for dividends < 2^31.  Grids are indexed with 32-bit
// linear indices per device (101^4 = 1.04e8 < 2^31).
struct FastDiv {
  uint32_t div;
  uint32_t mul;
  uint32_t shr;

  __host__ void init(uint32_t d) {
    div = d;
    if (d == 1) {
      mul = 0;
      shr = 0;
      return;
    }
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;  // ceil(log2 d)
    const uint64_t p = 31 + l;
    mul = static_cast<uint32_t>(((1ull << p) + d - 1) / d);
    shr = static_cast<uint32_t>(p - 32);
  }
  __device__ __forceinline__ uint32_t quo(uint32_t x) const {
    return mul == 0 ? x : (__umulhi(x, mul) >> shr);
  }
};

// godunov_flux (solver.cpp:44-63), the reference's Godunov numerical flux of
// one axis from the row's slopes and the one-sided differences
__device__ __forceinline__ double godunov_flux(double pos, double neg, double dminus,
                                               double dplus) {
  const double ha = dminus > 0.0 ? pos * dminus : neg * dminus;
  const double hb = dplus > 0.0 ? pos * dplus : neg * dplus;
  if (dminus <= dplus) {
    double h = ha > hb ? ha : hb;
    if (dminus <= 0.0 && 0.0 <= dplus && h < 0.0) h = 0.0;
    return h;
  }
  double h = ha < hb ? ha : hb;
  if (dplus <= 0.0 && 0.0 <= dminus && h > 0.0) h = 0.0;
  return h;
}

// Grid as the kernels see it: reference Grid (grid.hpp:23-48), strides last
// axis fastest, 1/spacing computed on the host (solver.cpp:208-209).
struct DevGrid {
  int nd;
  uint32_t size;
  uint32_t n[kMaxDims];
  uint32_t stride[kMaxDims];
  FastDiv divs[kMaxDims];  // divs[d] divides by n[d]
  double min[kMaxDims];
  double max[kMaxDims];
  double spacing[kMaxDims];
  double inv_spacing[kMaxDims];
};

// One state row of the separable affine model as the stencil consumes it.
//   folded: Godunov slopes pos/neg tabulated over one axis (constant
//           disturbance bounds): pos = tab[off_pos + k], neg = tab[off_neg + k]
//   else:   drift = tab[off_a + k_a] (+ tab[off_b + k_b]); then the
//           non-zero control/disturbance addends in reference order
//           (dim_slopes, solver.cpp:67-86).
struct DevRow {
  int folded;
  int axis_a, axis_b;    // -1: absent
  int off_a, off_b;      // table offsets of drift terms (non-folded)
  int off_pos, off_neg;  // folded Godunov slope tables
  int off_alpha;         // LF: alpha table over axis_a (-1: compute per node)
  int n_uadd;            // non-zero control terms of this row
  int uch[kMaxInput];
  double ucoef[kMaxInput];
  double uadd_pos[kMaxInput], uadd_neg[kMaxInput];  // min/max of B*ulo, B*uhi
  double ulo_term[kMaxInput], uhi_term[kMaxInput];  // flow_bounds min/max
  int n_dterm;           // non-zero disturbance coefficients of this row
  int dch[kMaxInput];
  double dcoef[kMaxInput];
  int constant_drift;    // drift has no coordinate term (axis_a == -1)
  double drift_const;
};

struct DevModel {
  int n, m, p;
  int per_node;
  DevRow row[kMaxDims];
  // LF: control / disturbance coefficient columns (non-zero entries only)
  int u_nrow[kMaxInput];
  int u_rows[kMaxInput][kMaxDims];
  double u_coef[kMaxInput][kMaxDims];
  double ulo[kMaxInput], uhi[kMaxInput];
  int d_nrow[kMaxInput];
  int d_rows[kMaxInput][kMaxDims];
  double d_coef[kMaxInput][kMaxDims];
  double dlo[kMaxInput], dhi[kMaxInput];  // constant bounds
  const double* tab;                      // device table storage
  const double* db_lo[kMaxInput];         // per-node bounds (device)
  const double* db_hi[kMaxInput];
};

// Device-side state of the iteration loop (solver.cpp:339-370), updated by
// the last CTA of every sweep.
struct LoopState {
  unsigned long long maxdv_bits;  // running max |dV| of the current sweep
  unsigned int blocks_done;
  unsigned int work_next;  // dynamic work-item counter of the persistent 4D sweep
  int done;
  int status;  // 0 ok, HJB_ERR_DIVERGED
  int converged;
  long long iter;
  long long max_iters;
  long long history_cap;
  double dt;
  double tol;
  double horizon;
  double min_residual;
  double first_residual;
  double last_residual;
  unsigned long long t0_ns;
  double* history;
  double* wall_history;
  // pipelined sharded loop: sweep k accumulates into maxdv_slot[k & 1] while
  // the all-reduce + epilogue of sweep k - 1 run on the comm stream
  unsigned long long maxdv_slot[2];
  unsigned int gen;  // grid-barrier generation of the multi-sweep kernel
  // sharded slab launches: finished boundary items (per consumer warp) and
  // the flag the halo transfer waits for (reset by the transfer stream)
  unsigned int bnd_done;
  unsigned int bnd_flag;
};

}  // namespace hjb
