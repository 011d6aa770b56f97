// hjb_kernels.cu — generic-rank sm_100a kernels of the HJ reachability solver.
//
// Bitwise contract: every expression below reproduces the reference's
// (proj/src/solver.cpp, dynamics.cpp, grid.cpp, levelset.cpp) operand order;
// built with -fmad=false no multiply-add is contracted.  Terms the reference
// accumulates with a zero coefficient (0*lo, 0*u) are skipped: adding +-0
// never changes a value, only possibly the sign of an exact zero, and the
// parity contract compares fields with IEEE ==.
#include <cuda_runtime.h>

#include <cstdint>

#include "hjb_kernels.cuh"

namespace hjb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int ND>
__device__ __forceinline__ void unravel(const DevGrid& g, uint32_t lin, uint32_t* idx) {
#pragma unroll
  for (int d = ND - 1; d >= 0; --d) {
    const uint32_t q = g.divs[d].quo(lin);
    idx[d] = lin - q * g.n[d];
    lin = q;
  }
}

// max over non-negative doubles through their IEEE bit patterns (which order
// like the values); NaN never enters: callers only fold values with `>`.
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v) {
  __shared__ unsigned long long part[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max_u64(v);
  if (lane == 0) part[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? part[lane] : 0ull;
    v = warp_max_u64(v);
  }
  return v;  // valid in thread 0
}

// Epilogue of one sweep: residual, histories, convergence and divergence
// tests of solver.cpp:347-369, executed by the last CTA to finish.
__device__ void finish_sweep(const StepArgs& a, double local_max) {
  LoopState* st = a.st;
  const unsigned long long b = block_max_u64(__double_as_longlong(local_max));
  if (threadIdx.x != 0) return;
  if (b) atomicMax(&st->maxdv_bits, b);
  if (!a.loop) return;
  __threadfence();
  const unsigned int ticket = atomicAdd(&st->blocks_done, 1u);
  if (ticket != gridDim.x * gridDim.y - 1) return;
  __threadfence();
  const unsigned long long bits = atomicAdd(&st->maxdv_bits, 0ull);
  const double max_dv = __longlong_as_double(bits);
  const double residual = max_dv / st->dt;
  const long long iter = st->iter + 1;
  st->iter = iter;
  if (iter - 1 < st->history_cap) {
    if (st->history) st->history[iter - 1] = residual;
    if (st->wall_history)
      st->wall_history[iter - 1] = (double)(globaltimer_ns() - st->t0_ns) * 1e-6;
  }
  st->last_residual = residual;
  bool stop = false;
  if (residual < st->tol) {
    st->converged = 1;
    stop = true;
  } else {
    if (iter == 1) st->first_residual = residual;
    const double mr0 = st->min_residual;
    const double mr = residual < mr0 ? residual : mr0;  // std::min(min_residual, residual)
    st->min_residual = mr;
    const double first = st->first_residual;
    const double base = mr < first ? first : mr;  // std::max(min_residual, front)
    if (!isfinite(residual) || residual > 10.0 * base) {
      st->status = HJB_ERR_DIVERGED;
      stop = true;
    }
  }
  if (iter >= st->max_iters) stop = true;
  if (st->horizon > 0.0 && (double)iter * st->dt >= st->horizon) stop = true;
  st->maxdv_bits = 0ull;
  st->blocks_done = 0u;
  st->work_next = 0u;
  if (stop) {
    st->done = 1;
    if (a.use_handle) cudaGraphSetConditional(a.handle, 0u);
  }
  __threadfence();
}

// drift_i(x) of the separable affine model (AffineFlow::drift, model
// affine() of dynamics.cpp:126-198 evaluated through host-built tables).
template <int ND>
__device__ __forceinline__ double row_drift(const DevModel& m, const DevRow& r,
                                            const uint32_t* idx) {
  if (r.constant_drift) return r.drift_const;
  double v = __ldg(m.tab + r.off_a + idx[r.axis_a]);
  if (r.axis_b >= 0) v = v + __ldg(m.tab + r.off_b + idx[r.axis_b]);
  return v;
}

template <bool PERNODE>
__device__ __forceinline__ void dist_bounds(const DevModel& m, int ch, uint32_t lin, double& lo,
                                            double& hi) {
  if (PERNODE) {
    lo = __ldg(m.db_lo[ch] + lin);
    hi = __ldg(m.db_hi[ch] + lin);
  } else {
    lo = m.dlo[ch];
    hi = m.dhi[ch];
  }
}

// dim_slopes for one row (solver.cpp:67-86)
template <int ND, bool PERNODE>
__device__ __forceinline__ void row_slopes(const DevModel& m, const DevRow& r,
                                           const uint32_t* idx, uint32_t lin, double& pos,
                                           double& neg) {
  if (!PERNODE && r.folded) {
    const uint32_t k = r.axis_a >= 0 ? idx[r.axis_a] : 0u;
    pos = __ldg(m.tab + r.off_pos + k);
    neg = __ldg(m.tab + r.off_neg + k);
    return;
  }
  const double dr = row_drift<ND>(m, r, idx);
  pos = dr;
  neg = dr;
  for (int t = 0; t < r.n_uadd; ++t) {
    pos += r.uadd_pos[t];
    neg += r.uadd_neg[t];
  }
  for (int t = 0; t < r.n_dterm; ++t) {
    double lo, hi;
    dist_bounds<PERNODE>(m, r.dch[t], lin, lo, hi);
    const double a = r.dcoef[t] * lo;
    const double b = r.dcoef[t] * hi;
    pos += a > b ? a : b;
    neg += a < b ? a : b;
  }
}

// godunov_flux (solver.cpp:44-63): hjb_device.cuh

// flow_bounds alpha for one row (dynamics.cpp:93-112)
template <int ND, bool PERNODE>
__device__ __forceinline__ double row_alpha(const DevModel& m, const DevRow& r,
                                            const uint32_t* idx, uint32_t lin) {
  if (!PERNODE && r.off_alpha >= 0) {
    const uint32_t k = r.axis_a >= 0 ? idx[r.axis_a] : 0u;
    return __ldg(m.tab + r.off_alpha + k);
  }
  const double dr = row_drift<ND>(m, r, idx);
  double lo = dr, hi = dr;
  for (int t = 0; t < r.n_uadd; ++t) {
    lo += r.ulo_term[t];
    hi += r.uhi_term[t];
  }
  for (int t = 0; t < r.n_dterm; ++t) {
    double dlo, dhi;
    dist_bounds<PERNODE>(m, r.dch[t], lin, dlo, dhi);
    const double a = r.dcoef[t] * dlo;
    const double b = r.dcoef[t] * dhi;
    lo += b < a ? b : a;  // std::min
    hi += a < b ? b : a;  // std::max
  }
  const double al = fabs(lo), ah = fabs(hi);
  return al < ah ? ah : al;
}

// extremal_inputs + hamiltonian (dynamics.cpp:37-83)
template <int ND, bool PERNODE>
__device__ __forceinline__ double lf_hamiltonian(const DevModel& m, const double* p,
                                                 const uint32_t* idx, uint32_t lin) {
  double u[kMaxInput], d[kMaxInput];
  for (int j = 0; j < m.m; ++j) {
    double coeff = 0.0;
    for (int t = 0; t < m.u_nrow[j]; ++t) coeff += p[m.u_rows[j][t]] * m.u_coef[j][t];
    u[j] = coeff > 0.0 ? m.ulo[j] : (coeff < 0.0 ? m.uhi[j] : m.ulo[j]);
  }
  for (int k = 0; k < m.p; ++k) {
    double coeff = 0.0;
    for (int t = 0; t < m.d_nrow[k]; ++t) coeff += p[m.d_rows[k][t]] * m.d_coef[k][t];
    double lo, hi;
    dist_bounds<PERNODE>(m, k, lin, lo, hi);
    d[k] = coeff > 0.0 ? hi : (coeff < 0.0 ? lo : lo);
  }
  double h = 0.0;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    const DevRow& r = m.row[i];
    double fi = row_drift<ND>(m, r, idx);
    for (int t = 0; t < r.n_uadd; ++t) fi += r.ucoef[t] * u[r.uch[t]];
    for (int t = 0; t < r.n_dterm; ++t) fi += r.dcoef[t] * d[r.dch[t]];
    h += p[i] * fi;
  }
  return h;
}

// K2/K3: update_chunk (solver.cpp:106-190) for one node per thread.
template <int ND, int SCHEME, bool PERNODE>
__global__ void __launch_bounds__(kThreads) k_step(const __grid_constant__ StepArgs a) {
  const double* src;
  double* dst;
  if (a.loop) {
    if (*(volatile int*)&a.st->done) return;
    const long long it = a.st->iter;
    src = (it & 1) ? a.buf1 : a.buf0;
    dst = (it & 1) ? a.buf0 : a.buf1;
  } else {
    src = a.src;
    dst = a.dst;
  }
  const DevGrid& g = a.g;
  double local = 0.0;
  for (uint32_t lin = blockIdx.x * blockDim.x + threadIdx.x; lin < g.size;
       lin += gridDim.x * blockDim.x) {
    uint32_t idx[ND];
    unravel<ND>(g, lin, idx);
    const double v = src[lin];
    double dm[ND], dp[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const uint32_t s = g.stride[d];
      const uint32_t k = idx[d];
      const double inv = g.inv_spacing[d];
      double left, right;
      if (k > 0 && k < g.n[d] - 1) {
        left = (v - src[lin - s]) * inv;
        right = (src[lin + s] - v) * inv;
      } else if (k == 0) {
        right = (src[lin + s] - v) * inv;
        left = SCHEME == kGodunov ? 0.0 : right;
      } else {
        left = (v - src[lin - s]) * inv;
        right = SCHEME == kGodunov ? 0.0 : left;
      }
      dm[d] = left;
      dp[d] = right;
    }
    double hhat = 0.0;
    if (SCHEME == kGodunov) {
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        double pos, neg;
        row_slopes<ND, PERNODE>(a.m, a.m.row[d], idx, lin, pos, neg);
        hhat += godunov_flux(pos, neg, dm[d], dp[d]);
      }
    } else {
      double p[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) p[d] = 0.5 * (dm[d] + dp[d]);
      hhat = lf_hamiltonian<ND, PERNODE>(a.m, p, idx, lin);
      if (SCHEME == kLfPerNode) {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          const double al = row_alpha<ND, PERNODE>(a.m, a.m.row[d], idx, lin);
          hhat += al * 0.5 * (dp[d] - dm[d]);
        }
      } else {
#pragma unroll
        for (int d = 0; d < ND; ++d) hhat += a.galpha[d] * 0.5 * (dp[d] - dm[d]);
      }
    }
    double stepped = v + a.dt * hhat;
    if (a.target) {  // std::min(stepped, l), then the reference clamp
      const double l = a.target[lin];
      stepped = l < stepped ? l : stepped;
    }
    const double cc = a.c[lin];
    const double vnew = stepped > cc ? stepped : cc;
    dst[lin] = vnew;
    const double dv = fabs(vnew - v);
    if (dv > local) local = dv;
  }
  finish_sweep(a, local);
}

// ---------------------------------------------------------------- K6
// ENO2/ENO3 + TVD-RK stages.  No reference; the definitions are
// the repo's CPU restatement's (oracle/hj_oracle.c, "high order" section),
// reproduced operation for operation.
constexpr double kThird = 1.0 / 3.0;
constexpr double kTwoThirds = 2.0 / 3.0;
constexpr double kSixthNeg = -1.0 / 6.0;

__device__ __forceinline__ double minabs(double x, double y) { return fabs(x) <= fabs(y) ? x : y; }

// face difference a(j) = (V[j+1] - V[j]) * inv along one axis; ghost faces:
// Godunov 0.0, LF the nearest interior face
template <bool GODUNOV>
__device__ __forceinline__ double face(const double* __restrict__ v, uint32_t lin, uint32_t stride,
                                       int k, int n, int j, double inv) {
  if (j < 0 || j > n - 2) {
    if (GODUNOV) return 0.0;
    j = j < 0 ? 0 : n - 2;
  }
  const double* p = v + lin + (long long)(j - k) * (long long)stride;
  return (p[stride] - p[0]) * inv;
}

template <bool GODUNOV>
__device__ __forceinline__ void eno_pair(const double* __restrict__ v, uint32_t lin,
                                         uint32_t stride, int k, int n, double inv, int ORDER,
                                         double& dm, double& dp) {
  if (ORDER <= 1) {
    dm = face<GODUNOV>(v, lin, stride, k, n, k - 1, inv);
    dp = face<GODUNOV>(v, lin, stride, k, n, k, inv);
    return;
  }
  double a[6];  // a(k-3) .. a(k+2)
#pragma unroll
  for (int t = 0; t < 6; ++t) a[t] = face<GODUNOV>(v, lin, stride, k, n, k - 3 + t, inv);
  // index helpers relative to k: A(j) = a[j - k + 3], D2(j) = A(j) - A(j-1)
#define A_(o) a[(o) + 3]
#define D2_(o) (A_(o) - A_((o)-1))
  if (ORDER == 2) {
    dm = A_(-1) + 0.5 * minabs(D2_(-1), D2_(0));
    dp = A_(0) + -0.5 * minabs(D2_(0), D2_(1));
  } else {
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int K = side == 0 ? -1 : 0;  // relative to k
      const double x = D2_(K), y = D2_(K + 1);
      const bool left = fabs(x) <= fabs(y);
      const double c2 = left ? x : y;
      const int ks = left ? K - 1 : K;
      double d3l, d3r;  // d3(ks), d3(ks+1)
      if (left) {
        d3l = D2_(K) - D2_(K - 1);
        d3r = D2_(K + 1) - D2_(K);
      } else {
        d3l = D2_(K + 1) - D2_(K);
        d3r = D2_(K + 2) - D2_(K + 1);
      }
      const double c3 = minabs(d3l, d3r);
      const int mm = -ks;  // k - ks
      const double w = mm == 1 ? kSixthNeg : kThird;
      const double s2 = side == 0 ? 0.5 : -0.5;
      const double d = (A_(K) + s2 * c2) + w * c3;
      if (side == 0) dm = d; else dp = d;
    }
  }
#undef D2_
#undef A_
}

template <int ND, int SCHEME, bool PERNODE>
__global__ void __launch_bounds__(kThreads) k_ho_stage(const __grid_constant__ StepArgs a) {
  if (a.loop && *(volatile int*)&a.st->done) return;
  const long long it = a.loop ? a.st->iter : 0;
  const double* vn = a.loop ? ((it & 1) ? a.buf1 : a.buf0) : a.src;
  double* outp = a.loop ? ((it & 1) ? a.buf0 : a.buf1) : a.dst;
  const double* vs = a.src_sel == 0 ? vn : (a.src_sel == 1 ? a.stage1 : a.stage2);
  double* dst = a.dst_sel == 0 ? outp : (a.dst_sel == 1 ? a.stage1 : a.stage2);
  const DevGrid& g = a.g;
  double local = 0.0;
  for (uint32_t lin = blockIdx.x * blockDim.x + threadIdx.x; lin < g.size;
       lin += gridDim.x * blockDim.x) {
    uint32_t idx[ND];
    unravel<ND>(g, lin, idx);
    double dm[ND], dp[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d)
      eno_pair<SCHEME == kGodunov>(vs, lin, g.stride[d], (int)idx[d], (int)g.n[d],
                                   g.inv_spacing[d], a.order, dm[d], dp[d]);
    double hhat = 0.0;
    if (SCHEME == kGodunov) {
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        double pos, neg;
        row_slopes<ND, PERNODE>(a.m, a.m.row[d], idx, lin, pos, neg);
        hhat += godunov_flux(pos, neg, dm[d], dp[d]);
      }
    } else {
      double p[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) p[d] = 0.5 * (dm[d] + dp[d]);
      hhat = lf_hamiltonian<ND, PERNODE>(a.m, p, idx, lin);
      if (SCHEME == kLfPerNode) {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          const double al = row_alpha<ND, PERNODE>(a.m, a.m.row[d], idx, lin);
          hhat += al * 0.5 * (dp[d] - dm[d]);
        }
      } else {
#pragma unroll
        for (int d = 0; d < ND; ++d) hhat += a.galpha[d] * 0.5 * (dp[d] - dm[d]);
      }
    }
    const double st = vs[lin] + a.dt * hhat;
    double val;
    switch (a.kind) {
      case 1: val = 0.5 * vn[lin] + 0.5 * st; break;
      case 2: val = 0.75 * vn[lin] + 0.25 * st; break;
      case 3: val = kThird * vn[lin] + kTwoThirds * st; break;
      default: val = st; break;
    }
    if (a.target) {  // every RK stage: min against the target, then the clamp
      const double l = a.target[lin];
      val = l < val ? l : val;
    }
    const double cc = a.c[lin];
    const double cl = val > cc ? val : cc;
    dst[lin] = cl;
    const double dv = fabs(cl - vn[lin]);
    if (dv > local) local = dv;
  }
  if (a.final_stage) finish_sweep(a, local);
}

// K1: scan_alpha (solver.cpp:221-268)
template <int ND, bool PERNODE>
__global__ void __launch_bounds__(kThreads) k_scan(const __grid_constant__ DevGrid g,
                                                   const __grid_constant__ DevModel m,
                                                   double* out) {
  const uint32_t lin = blockIdx.x * blockDim.x + threadIdx.x;
  double speed_max = 0.0;
  double amax[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) amax[d] = 0.0;
  if (lin < g.size) {
    uint32_t idx[ND];
    unravel<ND>(g, lin, idx);
    double speed = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const double al = row_alpha<ND, PERNODE>(m, m.row[d], idx, lin);
      speed += al * g.inv_spacing[d];
      amax[d] = al;
    }
    speed_max = speed;
  }
  unsigned long long b = block_max_u64(__double_as_longlong(speed_max));
  if (threadIdx.x == 0 && b) atomicMax((unsigned long long*)out, b);
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    __syncthreads();
    b = block_max_u64(__double_as_longlong(amax[d]));
    if (threadIdx.x == 0 && b) atomicMax((unsigned long long*)(out + 1 + d), b);
  }
}

__global__ void k_loop_init(LoopState* st, long long max_iters, double dt, double tol,
                            double horizon, long long history_cap, double* history,
                            double* wall_history) {
  st->maxdv_bits = 0ull;
  st->blocks_done = 0u;
  st->work_next = 0u;
  st->done = 0;
  st->status = 0;
  st->converged = 0;
  st->iter = 0;
  st->max_iters = max_iters;
  st->history_cap = history_cap;
  st->dt = dt;
  st->tol = tol;
  st->horizon = horizon;
  st->min_residual = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  st->first_residual = 0.0;
  st->last_residual = 0.0;
  st->history = history;
  st->wall_history = wall_history;
  st->maxdv_slot[0] = 0ull;
  st->maxdv_slot[1] = 0ull;
  st->gen = 0u;
  st->bnd_done = 0u;
  st->bnd_flag = 0u;
  st->t0_ns = globaltimer_ns();
}

// K4: resample (grid.cpp:84-135 locate/interp_ex, 215-231) with the optional
// seed clamp of solver.cpp:404-411.
template <int ND>
__global__ void __launch_bounds__(kThreads)
    k_resample(const __grid_constant__ DevGrid sg, const double* __restrict__ src,
               const __grid_constant__ DevGrid dg, double* __restrict__ dst,
               const double* slack, const double* __restrict__ c) {
  const uint32_t lin = blockIdx.x * blockDim.x + threadIdx.x;
  if (lin >= dg.size) return;
  uint32_t idx[ND];
  unravel<ND>(dg, lin, idx);
  uint32_t base[ND];
  double frac[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    const double x = idx[d] == dg.n[d] - 1 ? dg.max[d] : dg.min[d] + (double)idx[d] * dg.spacing[d];
    double t = (x - sg.min[d]) / sg.spacing[d];
    if (t < 0.0) t = 0.0;
    const double tmax = (double)(sg.n[d] - 1);
    if (t > tmax) t = tmax;
    uint32_t i0 = (uint32_t)t;
    if (i0 > sg.n[d] - 2) i0 = sg.n[d] - 2;
    base[d] = i0;
    frac[d] = t - (double)i0;
  }
  double value = 0.0;
  constexpr int corners = 1 << ND;
#pragma unroll 4
  for (int corner = 0; corner < corners; ++corner) {
    double w = 1.0;
    uint32_t l = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const bool hi = (corner >> d) & 1;
      w *= hi ? frac[d] : 1.0 - frac[d];
      l += (base[d] + (hi ? 1u : 0u)) * sg.stride[d];
    }
    if (w != 0.0) value += w * src[l];
  }
  if (c) {
    const double a = value - *slack;
    const double b = c[lin];
    value = a < b ? b : a;  // std::max(init - slack, constraint)
  }
  dst[lin] = value;
}

template <int ND>
__global__ void __launch_bounds__(kThreads)
    k_max_jump(const __grid_constant__ DevGrid g, const double* __restrict__ f, double* out) {
  const uint32_t lin = blockIdx.x * blockDim.x + threadIdx.x;
  double jump = 0.0;
  if (lin < g.size) {
    uint32_t idx[ND];
    unravel<ND>(g, lin, idx);
    const double v = f[lin];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      if (idx[d] + 1 >= g.n[d]) continue;
      const double dv = fabs(f[lin + g.stride[d]] - v);
      if (dv > jump) jump = dv;
    }
  }
  const unsigned long long b = block_max_u64(__double_as_longlong(jump));
  if (threadIdx.x == 0 && b) atomicMax((unsigned long long*)out, b);
}

template <int ND>
__global__ void k_band(const __grid_constant__ DevGrid g, int dim, double lo, double hi,
                       double* out) {
  const uint32_t lin = blockIdx.x * blockDim.x + threadIdx.x;
  if (lin >= g.size) return;
  uint32_t idx[ND];
  unravel<ND>(g, lin, idx);
  const uint32_t k = idx[dim];
  const double x = k == g.n[dim] - 1 ? g.max[dim] : g.min[dim] + (double)k * g.spacing[dim];
  const double a = lo - x, b = x - hi;
  out[lin] = a < b ? b : a;  // std::max(lo - x, x - hi)
}

__global__ void k_field_op(long long n, const double* __restrict__ a,
                           const double* __restrict__ b, double* __restrict__ out, int is_max) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double x = a[i];
    if (is_max == 2) {  // complement in level-set form: -f (exact)
      out[i] = -x;
      continue;
    }
    const double y = b[i];
    // std::max(x, y) / std::min(x, y) (levelset.cpp:80-86): ties keep x
    out[i] = is_max ? (x < y ? y : x) : (y < x ? y : x);
  }
}

__global__ void k_fill(double* out, uint32_t n, double value) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = value;
}

__global__ void k_not_constant(const double* __restrict__ f, uint32_t n, unsigned int* flag) {
  const unsigned long long first = __double_as_longlong(f[0]);
  bool diff = false;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    diff |= (unsigned long long)__double_as_longlong(f[i]) != first;
  if (__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(flag, 1u);
}

// ------------------------------------------------------ small 2D grids
// The whole solve() loop of a small 2D grid (config 1: 101^2) in ONE launch:
// a thread-block cluster of up to 16 CTAs, each owning a band of axis-0 rows
// of V (double-buffered) and c in shared memory; rows of the neighbouring
// bands are read through distributed shared memory.  Per sweep: update, CTA
// max, every CTA publishes its max into rank 0's slots (double-buffered by
// sweep parity), one cluster barrier, then every CTA reduces the slots and
// applies the solve() loop logic (solver.cpp:347-369) redundantly (identical
// inputs, identical decisions); CTA 0 writes the histories.
struct Small2dArgs {
  StepArgs s;        // grid/model/c/dt/scheme/galpha; s.src = init, s.dst = out
  uint32_t rows;     // axis-0 rows per CTA (last CTA may own fewer)
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctas() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ const double* map_rank(const double* p, uint32_t rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<const double*>(out);
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

template <int SCHEME, bool PERNODE>
__global__ void __launch_bounds__(512, 1) k_small2d(const __grid_constant__ Small2dArgs a) {
  extern __shared__ __align__(16) double sm[];
  const StepArgs& p = a.s;
  const DevGrid& g = p.g;
  const uint32_t n0 = g.n[0], n1 = g.n[1];
  const uint32_t R = a.rows;
  const uint32_t me = cluster_ctarank(), nct = cluster_nctas();
  const uint32_t r0 = me * R;
  const uint32_t r1 = min(r0 + R, n0);
  const uint32_t own = r1 > r0 ? (r1 - r0) * n1 : 0;
  double* buf[2] = {sm, sm + R * n1};
  double* cl = sm + 2 * R * n1;
  unsigned long long* slots = reinterpret_cast<unsigned long long*>(sm + 3 * R * n1);  // [2][16]
  __shared__ unsigned long long part[32];
  __shared__ int s_done;
  for (uint32_t t = threadIdx.x; t < own; t += blockDim.x) {
    buf[0][t] = p.src[r0 * n1 + t];
    cl[t] = p.c[r0 * n1 + t];
  }
  const double inv0 = g.inv_spacing[0], inv1 = g.inv_spacing[1];
  // loop state (identical in every CTA)
  long long iter = 0;
  double min_res = __longlong_as_double(0x7ff0000000000000ll), first = 0.0, residual = 0.0;
  int converged = 0, status = 0;
  cluster_sync_all();
  const double* remote_prev[2];
  const double* remote_next[2];
  for (int b = 0; b < 2; ++b) {
    remote_prev[b] = me > 0 ? map_rank(buf[b], me - 1) : nullptr;
    remote_next[b] = me + 1 < nct ? map_rank(buf[b], me + 1) : nullptr;
  }
  unsigned long long* slots0 = const_cast<unsigned long long*>(
      reinterpret_cast<const unsigned long long*>(map_rank(reinterpret_cast<const double*>(slots), 0)));
  const unsigned long long t0 = globaltimer_ns();
  for (;;) {
    const int cb = static_cast<int>(iter & 1);
    const double* cur = buf[cb];
    double* nxt = buf[cb ^ 1];
    double local = 0.0;
    for (uint32_t t = threadIdx.x; t < own; t += blockDim.x) {
      const uint32_t lr = t / n1, k1 = t - lr * n1;
      const uint32_t k0 = r0 + lr;
      uint32_t idx[2] = {k0, k1};
      const uint32_t lin = k0 * n1 + k1;
      const double v = cur[t];
      // axis-0 neighbours: local rows or the neighbouring bands (DSMEM)
      double vm0 = 0.0, vp0 = 0.0;
      if (k0 > 0) vm0 = lr > 0 ? cur[t - n1] : remote_prev[cb][(R - 1) * n1 + k1];
      if (k0 + 1 < n0) vp0 = lr + 1 < r1 - r0 ? cur[t + n1] : remote_next[cb][k1];
      double dm[2], dp[2];
      // solver.cpp:134-151
      if (k0 > 0 && k0 < n0 - 1) {
        dm[0] = (v - vm0) * inv0;
        dp[0] = (vp0 - v) * inv0;
      } else if (k0 == 0) {
        dp[0] = (vp0 - v) * inv0;
        dm[0] = SCHEME == kGodunov ? 0.0 : dp[0];
      } else {
        dm[0] = (v - vm0) * inv0;
        dp[0] = SCHEME == kGodunov ? 0.0 : dm[0];
      }
      if (k1 > 0 && k1 < n1 - 1) {
        dm[1] = (v - cur[t - 1]) * inv1;
        dp[1] = (cur[t + 1] - v) * inv1;
      } else if (k1 == 0) {
        dp[1] = (cur[t + 1] - v) * inv1;
        dm[1] = SCHEME == kGodunov ? 0.0 : dp[1];
      } else {
        dm[1] = (v - cur[t - 1]) * inv1;
        dp[1] = SCHEME == kGodunov ? 0.0 : dm[1];
      }
      double hhat = 0.0;
      if (SCHEME == kGodunov) {
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          double pos, neg;
          row_slopes<2, PERNODE>(p.m, p.m.row[d], idx, lin, pos, neg);
          hhat += godunov_flux(pos, neg, dm[d], dp[d]);
        }
      } else {
        double q[2] = {0.5 * (dm[0] + dp[0]), 0.5 * (dm[1] + dp[1])};
        hhat = lf_hamiltonian<2, PERNODE>(p.m, q, idx, lin);
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          const double al = SCHEME == kLfPerNode ? row_alpha<2, PERNODE>(p.m, p.m.row[d], idx, lin)
                                                 : p.galpha[d];
          hhat += al * 0.5 * (dp[d] - dm[d]);
        }
      }
      const double stepped = v + p.dt * hhat;
      const double cc = cl[t];
      const double vnew = stepped > cc ? stepped : cc;
      nxt[t] = vnew;
      const double dv = fabs(vnew - v);
      if (dv > local) local = dv;
    }
    // CTA max -> slot of rank 0
    unsigned long long bm = warp_max_u64(__double_as_longlong(local));
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = bm;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0;
      for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) m = part[w] > m ? part[w] : m;
      slots0[cb * 16 + me] = m;
    }
    cluster_sync_all();
    if (threadIdx.x == 0) {
      unsigned long long m = 0;
      for (uint32_t r = 0; r < nct; ++r) {
        const unsigned long long x = slots0[cb * 16 + r];
        m = x > m ? x : m;
      }
      residual = __longlong_as_double(m) / p.dt;
      ++iter;
      LoopState* st = p.st;
      if (me == 0 && iter - 1 < st->history_cap) {
        if (st->history) st->history[iter - 1] = residual;
        if (st->wall_history)
          st->wall_history[iter - 1] = (double)(globaltimer_ns() - t0) * 1e-6;
      }
      bool stop = false;
      if (residual < p.st->tol) {
        converged = 1;
        stop = true;
      } else {
        if (iter == 1) first = residual;
        min_res = residual < min_res ? residual : min_res;
        const double base = min_res < first ? first : min_res;
        if (!isfinite(residual) || residual > 10.0 * base) {
          status = HJB_ERR_DIVERGED;
          stop = true;
        }
      }
      if (iter >= p.st->max_iters) stop = true;
      if (p.st->horizon > 0.0 && (double)iter * p.dt >= p.st->horizon) stop = true;
      s_done = stop ? 1 : 0;
    }
    __syncthreads();
    // every thread tracks iter identically (thread 0's value broadcast)
    if (threadIdx.x != 0) ++iter;
    if (s_done) break;
  }
  // write the final iterate (buffer parity of iter) and the loop state
  const double* fin = buf[iter & 1];
  for (uint32_t t = threadIdx.x; t < own; t += blockDim.x) p.dst[r0 * n1 + t] = fin[t];
  if (me == 0 && threadIdx.x == 0) {
    LoopState* st = p.st;
    st->iter = iter;
    st->converged = converged;
    st->status = status;
    st->last_residual = residual;
    st->done = 1;
  }
  cluster_sync_all();  // keep every CTA's shared memory alive until all DSMEM reads are done
}

// High-order (ENO1..3 + TVD-RK1..3) variant of k_small2d: every RK stage of
// every step in the same single cluster launch (BASELINE config 1 scheme:
// ENO2 + TVD-RK2 on 101^2).  Per CTA band of rows in shared memory: V_n
// (double-buffered by parity), stage1, stage2, c.  A stage reads its input
// rows of any band through DSMEM (mapa), writes its output band, and ends
// with a cluster barrier; the last stage of a step also reduces max|dV| and
// applies the solve() loop logic, as k_small2d.  The stencil arithmetic is
// eno_pair / godunov_flux / lf_hamiltonian, as k_ho_stage.
template <int SCHEME, bool PERNODE>
__global__ void __launch_bounds__(512, 1) k_small2d_ho(const __grid_constant__ Small2dArgs a) {
  extern __shared__ __align__(16) double sm[];
  const StepArgs& p = a.s;
  const DevGrid& g = p.g;
  const uint32_t n0 = g.n[0], n1 = g.n[1];
  const uint32_t RB = a.rows;  // rows per band
  const uint32_t me = cluster_ctarank(), nct = cluster_nctas();
  const uint32_t r0 = me * RB;
  const uint32_t r1 = min(r0 + RB, n0);
  const uint32_t own = r1 > r0 ? (r1 - r0) * n1 : 0;
  const uint32_t band = RB * n1;
  double* bufs[4] = {sm, sm + band, sm + 2 * band, sm + 3 * band};  // V even, V odd, s1, s2
  double* cl = sm + 4 * band;
  unsigned long long* slots = reinterpret_cast<unsigned long long*>(sm + 5 * band);  // [2][16]
  __shared__ unsigned long long part[32];
  __shared__ int s_done;
  for (uint32_t t = threadIdx.x; t < own; t += blockDim.x) {
    bufs[0][t] = p.src[r0 * n1 + t];
    cl[t] = p.c[r0 * n1 + t];
  }
  const double inv0 = g.inv_spacing[0], inv1 = g.inv_spacing[1];
  const int order = p.order;
  const int rk = p.kind;  // TVD-RK order (1..3), carried in StepArgs.kind for this kernel
  // stage table (src, dst, kind): buffers 0 = V_n, 1 = stage1, 2 = stage2, 3 = V_{n+1}
  int ns = 1, ssrc[3] = {0, 0, 0}, sdst[3] = {3, 3, 3}, skind[3] = {0, 0, 0};
  if (rk == 2) {
    ns = 2;
    sdst[0] = 1; ssrc[1] = 1; sdst[1] = 3; skind[1] = 1;
  } else if (rk >= 3) {
    ns = 3;
    sdst[0] = 1; ssrc[1] = 1; sdst[1] = 2; skind[1] = 2; ssrc[2] = 2; sdst[2] = 3; skind[2] = 3;
  }
  long long iter = 0;
  double min_res = __longlong_as_double(0x7ff0000000000000ll), first = 0.0, residual = 0.0;
  int converged = 0, status = 0;
  cluster_sync_all();
  unsigned long long* slots0 = const_cast<unsigned long long*>(
      reinterpret_cast<const unsigned long long*>(map_rank(reinterpret_cast<const double*>(slots), 0)));
  const unsigned long long t0 = globaltimer_ns();
  for (;;) {
    const int cb = static_cast<int>(iter & 1);
    double local = 0.0;
    for (int q = 0; q < ns; ++q) {
      const int sb = ssrc[q] == 0 ? cb : ssrc[q] + 1;  // smem buffer index of the input
      const int db = sdst[q] == 3 ? (cb ^ 1) : sdst[q] + 1;
      const double* in = bufs[sb];
      const double* vnb = bufs[cb];
      double* outb = bufs[db];
      const bool last = q == ns - 1;
      for (uint32_t t = threadIdx.x; t < own; t += blockDim.x) {
        const uint32_t lr = t / n1, k1 = t - lr * n1;
        const uint32_t k0 = r0 + lr;
        uint32_t idx[2] = {k0, k1};
        const uint32_t lin = k0 * n1 + k1;
        // axis-0 column k0-3 .. k0+3 of the stage input (any band, DSMEM)
        double col[7];
#pragma unroll
        for (int o = -3; o <= 3; ++o) {
          const int j = (int)k0 + o;
          double x = 0.0;
          if (j >= 0 && j < (int)n0 && (o >= -order && o <= order)) {
            const uint32_t owner = (uint32_t)j / RB;
            const uint32_t off = ((uint32_t)j - owner * RB) * n1 + k1;
            x = owner == me ? in[off] : map_rank(in, owner)[off];
          }
          col[o + 3] = x;
        }
        double dm[2], dp[2];
        eno_pair<SCHEME == kGodunov>(col, 3, 1, (int)k0, (int)n0, inv0, order, dm[0], dp[0]);
        eno_pair<SCHEME == kGodunov>(in + lr * n1, k1, 1, (int)k1, (int)n1, inv1, order, dm[1],
                                     dp[1]);
        double hhat = 0.0;
        if (SCHEME == kGodunov) {
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            double pos, neg;
            row_slopes<2, PERNODE>(p.m, p.m.row[d], idx, lin, pos, neg);
            hhat += godunov_flux(pos, neg, dm[d], dp[d]);
          }
        } else {
          double pq[2] = {0.5 * (dm[0] + dp[0]), 0.5 * (dm[1] + dp[1])};
          hhat = lf_hamiltonian<2, PERNODE>(p.m, pq, idx, lin);
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const double al = SCHEME == kLfPerNode
                                  ? row_alpha<2, PERNODE>(p.m, p.m.row[d], idx, lin)
                                  : p.galpha[d];
            hhat += al * 0.5 * (dp[d] - dm[d]);
          }
        }
        const double st = in[t] + p.dt * hhat;
        const double vn = vnb[t];
        double val;
        switch (skind[q]) {
          case 1: val = 0.5 * vn + 0.5 * st; break;
          case 2: val = 0.75 * vn + 0.25 * st; break;
          case 3: val = kThird * vn + kTwoThirds * st; break;
          default: val = st; break;
        }
        const double cc = cl[t];
        const double vnew = val > cc ? val : cc;
        outb[t] = vnew;
        if (last) {
          const double dv = fabs(vnew - vn);
          if (dv > local) local = dv;
        }
      }
      if (!last) cluster_sync_all();  // the next stage reads this output across bands
    }
    unsigned long long bm = warp_max_u64(__double_as_longlong(local));
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = bm;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m = 0;
      for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) m = part[w] > m ? part[w] : m;
      slots0[cb * 16 + me] = m;
    }
    cluster_sync_all();
    if (threadIdx.x == 0) {
      unsigned long long m = 0;
      for (uint32_t r = 0; r < nct; ++r) {
        const unsigned long long x = slots0[cb * 16 + r];
        m = x > m ? x : m;
      }
      residual = __longlong_as_double(m) / p.dt;
      ++iter;
      LoopState* st = p.st;
      if (me == 0 && iter - 1 < st->history_cap) {
        if (st->history) st->history[iter - 1] = residual;
        if (st->wall_history)
          st->wall_history[iter - 1] = (double)(globaltimer_ns() - t0) * 1e-6;
      }
      bool stop = false;
      if (residual < p.st->tol) {
        converged = 1;
        stop = true;
      } else {
        if (iter == 1) first = residual;
        min_res = residual < min_res ? residual : min_res;
        const double base = min_res < first ? first : min_res;
        if (!isfinite(residual) || residual > 10.0 * base) {
          status = HJB_ERR_DIVERGED;
          stop = true;
        }
      }
      if (iter >= p.st->max_iters) stop = true;
      if (p.st->horizon > 0.0 && (double)iter * p.dt >= p.st->horizon) stop = true;
      s_done = stop ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x != 0) ++iter;
    if (s_done) break;
  }
  const double* fin = bufs[iter & 1];
  for (uint32_t t = threadIdx.x; t < own; t += blockDim.x) p.dst[r0 * n1 + t] = fin[t];
  if (me == 0 && threadIdx.x == 0) {
    LoopState* st = p.st;
    st->iter = iter;
    st->converged = converged;
    st->status = status;
    st->last_residual = residual;
    st->done = 1;
  }
  cluster_sync_all();
}

inline dim3 blocks_for(uint32_t n) { return dim3((n + kThreads - 1) / kThreads); }

// Persistent-style grid: a few CTAs per SM stride over the nodes, so the
// per-sweep epilogue sees ~10^3 CTA arrivals instead of one per 256 nodes.
inline dim3 step_blocks(uint32_t n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const uint32_t want = (n + kThreads - 1) / kThreads;
  const uint32_t cap = static_cast<uint32_t>(sms) * 8u;
  return dim3(want < cap ? want : cap);
}

template <int ND>
cudaError_t step_nd(const StepArgs& a, cudaStream_t s) {
  const dim3 grid = step_blocks(a.g.size);
  const bool pn = a.m.per_node != 0;
  switch (a.scheme) {
    case kGodunov:
      if (pn) k_step<ND, kGodunov, true><<<grid, kThreads, 0, s>>>(a);
      else k_step<ND, kGodunov, false><<<grid, kThreads, 0, s>>>(a);
      break;
    case kLfPerNode:
      if (pn) k_step<ND, kLfPerNode, true><<<grid, kThreads, 0, s>>>(a);
      else k_step<ND, kLfPerNode, false><<<grid, kThreads, 0, s>>>(a);
      break;
    default:
      if (pn) k_step<ND, kLfGlobal, true><<<grid, kThreads, 0, s>>>(a);
      else k_step<ND, kLfGlobal, false><<<grid, kThreads, 0, s>>>(a);
      break;
  }
  return cudaGetLastError();
}

}  // namespace

#define HJB_DISPATCH_ND(nd, CALL) \
  switch (nd) {                    \
    case 1: CALL(1); break;        \
    case 2: CALL(2); break;        \
    case 3: CALL(3); break;        \
    case 4: CALL(4); break;        \
    case 5: CALL(5); break;        \
    case 6: CALL(6); break;        \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_step(const StepArgs& a, cudaStream_t s) {
#define CALL(N) return step_nd<N>(a, s)
  HJB_DISPATCH_ND(a.g.nd, CALL)
#undef CALL
  return cudaSuccess;
}

template <int ND>
cudaError_t ho_nd(const StepArgs& a, cudaStream_t s) {
  const dim3 grid = step_blocks(a.g.size);
  const bool pn = a.m.per_node != 0;
  switch (a.scheme) {
    case kGodunov:
      if (pn) k_ho_stage<ND, kGodunov, true><<<grid, kThreads, 0, s>>>(a);
      else k_ho_stage<ND, kGodunov, false><<<grid, kThreads, 0, s>>>(a);
      break;
    case kLfPerNode:
      if (pn) k_ho_stage<ND, kLfPerNode, true><<<grid, kThreads, 0, s>>>(a);
      else k_ho_stage<ND, kLfPerNode, false><<<grid, kThreads, 0, s>>>(a);
      break;
    default:
      if (pn) k_ho_stage<ND, kLfGlobal, true><<<grid, kThreads, 0, s>>>(a);
      else k_ho_stage<ND, kLfGlobal, false><<<grid, kThreads, 0, s>>>(a);
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_ho_stage(const StepArgs& a, cudaStream_t s) {
  switch (a.g.nd) {
    case 1: return ho_nd<1>(a, s);
    case 2: return ho_nd<2>(a, s);
    case 3: return ho_nd<3>(a, s);
    case 4: return ho_nd<4>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_scan(const DevGrid& g, const DevModel& m, double* out, cudaStream_t s) {
  const dim3 grid = blocks_for(g.size);
#define CALL(N)                                                    \
  if (m.per_node) k_scan<N, true><<<grid, kThreads, 0, s>>>(g, m, out); \
  else k_scan<N, false><<<grid, kThreads, 0, s>>>(g, m, out)
  HJB_DISPATCH_ND(g.nd, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_loop_init(LoopState* st, long long max_iters, double dt, double tol,
                             double horizon, long long history_cap, double* history,
                             double* wall_history, cudaStream_t s) {
  k_loop_init<<<1, 1, 0, s>>>(st, max_iters, dt, tol, horizon, history_cap, history,
                              wall_history);
  return cudaGetLastError();
}

cudaError_t launch_resample(const DevGrid& sg, const double* src, const DevGrid& dg,
                            double* dst, const double* slack, const double* c,
                            cudaStream_t s) {
  const dim3 grid = blocks_for(dg.size);
#define CALL(N) k_resample<N><<<grid, kThreads, 0, s>>>(sg, src, dg, dst, slack, c)
  HJB_DISPATCH_ND(dg.nd, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_max_adjacent_jump(const DevGrid& g, const double* f, double* out,
                                     cudaStream_t s) {
  const dim3 grid = blocks_for(g.size);
#define CALL(N) k_max_jump<N><<<grid, kThreads, 0, s>>>(g, f, out)
  HJB_DISPATCH_ND(g.nd, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_band(const DevGrid& g, int dim, double lo, double hi, double* out,
                        cudaStream_t s) {
  const dim3 grid = blocks_for(g.size);
#define CALL(N) k_band<N><<<grid, kThreads, 0, s>>>(g, dim, lo, hi, out)
  HJB_DISPATCH_ND(g.nd, CALL)
#undef CALL
  return cudaGetLastError();
}

cudaError_t launch_fill(double* out, uint32_t n, double value, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint32_t b = (n + kThreads - 1) / kThreads;
  k_fill<<<b < 148 * 16 ? b : 148 * 16, kThreads, 0, s>>>(out, n, value);
  return cudaGetLastError();
}

cudaError_t launch_not_constant(const double* f, uint32_t n, unsigned int* flag, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint32_t b = (n + kThreads - 1) / kThreads;
  k_not_constant<<<b < 148 * 8 ? b : 148 * 8, kThreads, 0, s>>>(f, n, flag);
  return cudaGetLastError();
}

// flag := 1 if f[lin] differs (bit pattern) from f at the first node of its
// axis-0 plane, i.e. the field is not a function of i0 alone
__global__ void k_not_axis0(const double* __restrict__ f, uint32_t n, uint32_t s0,
                            unsigned int* flag) {
  for (uint32_t lin = blockIdx.x * blockDim.x + threadIdx.x; lin < n;
       lin += gridDim.x * blockDim.x) {
    const uint32_t base = lin - lin % s0;
    if (__double_as_longlong(f[lin]) != __double_as_longlong(f[base])) {
      *flag = 1u;
      return;
    }
  }
}

cudaError_t launch_not_axis0(const double* f, uint32_t n, uint32_t s0, unsigned int* flag,
                             cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint32_t b = (n + kThreads - 1) / kThreads;
  k_not_axis0<<<b < 148 * 8 ? b : 148 * 8, kThreads, 0, s>>>(f, n, s0, flag);
  return cudaGetLastError();
}

size_t small2d_smem(const DevGrid& g, uint32_t* rows_out, uint32_t* ctas_out) {
  if (g.nd != 2) return 0;
  const uint32_t R = (g.n[0] + 15) / 16;
  const uint32_t nct = (g.n[0] + R - 1) / R;
  if (rows_out) *rows_out = R;
  if (ctas_out) *ctas_out = nct;
  return (3ull * R * g.n[1]) * sizeof(double) + 32 * sizeof(unsigned long long);
}

size_t small2d_ho_smem(const DevGrid& g, uint32_t* rows_out, uint32_t* ctas_out) {
  if (g.nd != 2) return 0;
  const uint32_t R = (g.n[0] + 15) / 16;
  const uint32_t nct = (g.n[0] + R - 1) / R;
  if (rows_out) *rows_out = R;
  if (ctas_out) *ctas_out = nct;
  return (5ull * R * g.n[1]) * sizeof(double) + 32 * sizeof(unsigned long long);
}

cudaError_t launch_small2d_ho(const StepArgs& s, int rk, cudaStream_t stream) {
  uint32_t R = 0, nct = 0;
  const size_t smem = small2d_ho_smem(s.g, &R, &nct);
  Small2dArgs a;
  a.s = s;
  a.s.kind = rk;
  a.rows = R;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nct);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = nct;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return cudaLaunchKernelEx(&cfg, kernel, a);
  };
  const bool pn = s.m.per_node != 0;
  switch (s.scheme) {
    case kGodunov: return pn ? go(k_small2d_ho<kGodunov, true>) : go(k_small2d_ho<kGodunov, false>);
    case kLfPerNode:
      return pn ? go(k_small2d_ho<kLfPerNode, true>) : go(k_small2d_ho<kLfPerNode, false>);
    default: return pn ? go(k_small2d_ho<kLfGlobal, true>) : go(k_small2d_ho<kLfGlobal, false>);
  }
}

cudaError_t launch_small2d(const StepArgs& s, cudaStream_t stream) {
  uint32_t R = 0, nct = 0;
  const size_t smem = small2d_smem(s.g, &R, &nct);
  Small2dArgs a;
  a.s = s;
  a.rows = R;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nct);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = nct;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return cudaLaunchKernelEx(&cfg, kernel, a);
  };
  const bool pn = s.m.per_node != 0;
  switch (s.scheme) {
    case kGodunov: return pn ? go(k_small2d<kGodunov, true>) : go(k_small2d<kGodunov, false>);
    case kLfPerNode:
      return pn ? go(k_small2d<kLfPerNode, true>) : go(k_small2d<kLfPerNode, false>);
    default: return pn ? go(k_small2d<kLfGlobal, true>) : go(k_small2d<kLfGlobal, false>);
  }
}

cudaError_t launch_field_op(long long n, const double* a, const double* b, double* out,
                            int is_max, cudaStream_t s) {
  const int blocks = (int)((n + kThreads - 1) / kThreads < 148 * 16 ? (n + kThreads - 1) / kThreads
                                                                     : 148 * 16);
  if (n <= 0) return cudaSuccess;
  k_field_op<<<blocks, kThreads, 0, s>>>(n, a, b, out, is_max);
  return cudaGetLastError();
}

}  // namespace hjb
