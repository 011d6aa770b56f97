// hjb_filter.cu — batched SafetyFilter queries on the device.
//
// One thread per query state x: the reference's per-query work
// (safety.cpp:86-127) restated with the same arithmetic in the same order:
//   interp_ex(V, x)              grid.cpp:90-131 (locate + multilinear corners,
//                                `if (w != 0.0) value += w * field[lin]`)
//   max_cell_jump(V, x)          grid.cpp:177-195 (filter mode only)
//   interpolated_costate(V, x)   safety.cpp:14-49 with gradient_at,
//                                grid.cpp:141-163
//   IntervalField::at(ch, x)     interval_field.cpp:29-31 (multilinear of the
//                                lo / hi fields; a constant field is
//                                interpolated node by node like the reference)
//   extremal_inputs              dynamics.cpp:37-63 (bang-bang control,
//                                ties to lo; maximising disturbance)
// The value function stays in HBM; each query gathers 2^nd corners plus
// their axis neighbours, so the batch is latency-bound gather work — one
// warp covers 32 independent queries.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "hjb_internal.cuh"

namespace hjb {

namespace {

struct FilterArgs {
  DevGrid g;
  int n, m, p;
  int per_node;
  double B[kMaxState][kMaxInput];
  double C[kMaxState][kMaxInput];
  double ulo[kMaxInput], uhi[kMaxInput];
  double dlo_c[kMaxInput], dhi_c[kMaxInput];
  const double* dlo[kMaxInput];
  const double* dhi[kMaxInput];
  const double* V;
  long long nq;
  const double* x;
  const double* u_perf;
  int mode;
  double eta_floor, lambda;
  double* o_value;
  double* o_band;
  double* o_control;
  double* o_worst;
  uint8_t* o_flags;
  unsigned int* err;
};

template <int ND>
__global__ void __launch_bounds__(128) k_filter(const __grid_constant__ FilterArgs a) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= a.nq) return;
  const DevGrid& g = a.g;
  double xq[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) xq[d] = a.x[q * ND + d];
  // locate (grid.cpp:90-111); interpolated_costate's own locate
  // (safety.cpp:21-30) clamps to the same base / frac without the flag
  uint32_t base[ND];
  double frac[ND];
  bool ood = false;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    if (!isfinite(xq[d])) {
      atomicOr(a.err, 1u);
      return;
    }
    double t = (xq[d] - g.min[d]) / g.spacing[d];
    if (t < 0.0) {
      t = 0.0;
      ood = true;
    }
    const double tmax = (double)(g.n[d] - 1);
    if (t > tmax) {
      t = tmax;
      if (xq[d] > g.max[d]) ood = true;
    }
    uint32_t i0 = (uint32_t)t;
    if (i0 > g.n[d] - 2) i0 = g.n[d] - 2;
    base[d] = i0;
    frac[d] = t - (double)i0;
  }
  constexpr int corners = 1 << ND;
  // interp_ex (grid.cpp:113-131)
  double value = 0.0;
  for (int corner = 0; corner < corners; ++corner) {
    double w = 1.0;
    uint32_t lin = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const bool hi = (corner >> d) & 1;
      w *= hi ? frac[d] : 1.0 - frac[d];
      lin += (base[d] + (hi ? 1u : 0u)) * g.stride[d];
    }
    if (w != 0.0) value += w * __ldg(a.V + lin);
  }

  double band = 0.0;
  if (a.mode == HJB_FILTER_FILTER) {
    // max_cell_jump (grid.cpp:177-195)
    double jump = 0.0;
    for (int corner = 0; corner < corners; ++corner) {
      uint32_t lin = 0;
#pragma unroll
      for (int d = 0; d < ND; ++d) lin += (base[d] + ((corner >> d) & 1)) * g.stride[d];
      const double v0 = __ldg(a.V + lin);
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        if ((corner >> d) & 1) continue;
        const double dv = fabs(__ldg(a.V + lin + g.stride[d]) - v0);
        if (dv > jump) jump = dv;
      }
    }
    const double half = 0.5 * jump;
    const double eta = a.eta_floor < half ? half : a.eta_floor;  // std::max(eta_floor, ...)
    band = eta;
    if (!ood && value <= -a.lambda - eta) {  // safety.cpp:115-123: pass through
      if (a.o_value) a.o_value[q] = value;
      if (a.o_band) a.o_band[q] = eta;
      if (a.o_control)
        for (int j = 0; j < a.m; ++j) a.o_control[q * a.m + j] = a.u_perf[q * a.m + j];
      if (a.o_worst)
        for (int k = 0; k < a.p; ++k) a.o_worst[q * a.p + k] = 0.0;
      if (a.o_flags) a.o_flags[q] = 0;
      return;
    }
  }

  // interpolated_costate (safety.cpp:14-49)
  double costate[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) costate[d] = 0.0;
  double dlo[kMaxInput], dhi[kMaxInput];
  for (int k = 0; k < a.p; ++k) {
    dlo[k] = 0.0;
    dhi[k] = 0.0;
  }
  for (int corner = 0; corner < corners; ++corner) {
    double w = 1.0;
    uint32_t lin = 0;
    uint32_t kk[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const bool hi = (corner >> d) & 1;
      w *= hi ? frac[d] : 1.0 - frac[d];
      kk[d] = base[d] + (hi ? 1u : 0u);
      lin += kk[d] * g.stride[d];
    }
    if (w == 0.0) continue;
    const double f0 = __ldg(a.V + lin);
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      // gradient_at (grid.cpp:141-163): replicate the one-sided value at an edge
      const uint32_t s = g.stride[d];
      double left, right;
      if (kk[d] > 0 && kk[d] < g.n[d] - 1) {
        left = (f0 - __ldg(a.V + lin - s)) * g.inv_spacing[d];
        right = (__ldg(a.V + lin + s) - f0) * g.inv_spacing[d];
      } else if (kk[d] == 0) {
        right = (__ldg(a.V + lin + s) - f0) * g.inv_spacing[d];
        left = right;
      } else {
        left = (f0 - __ldg(a.V + lin - s)) * g.inv_spacing[d];
        right = left;
      }
      costate[d] += w * 0.5 * (left + right);
    }
    // IntervalField::at: interp of the lo / hi fields (same corners, same w)
    for (int k = 0; k < a.p; ++k) {
      const double lo = a.per_node ? __ldg(a.dlo[k] + lin) : a.dlo_c[k];
      const double hi = a.per_node ? __ldg(a.dhi[k] + lin) : a.dhi_c[k];
      dlo[k] += w * lo;
      dhi[k] += w * hi;
    }
  }

  // extremal_inputs (dynamics.cpp:37-63)
  bool any_active = false;
  for (int j = 0; j < a.m; ++j) {
    double coeff = 0.0;
    for (int i = 0; i < a.n; ++i) coeff += costate[i] * a.B[i][j];
    const double u = coeff > 0.0 ? a.ulo[j] : (coeff < 0.0 ? a.uhi[j] : a.ulo[j]);
    if (coeff != 0.0) any_active = true;
    if (a.o_control) a.o_control[q * a.m + j] = u;
  }
  for (int k = 0; k < a.p; ++k) {
    double coeff = 0.0;
    for (int i = 0; i < a.n; ++i) coeff += costate[i] * a.C[i][k];
    const double dk = coeff > 0.0 ? dhi[k] : (coeff < 0.0 ? dlo[k] : dlo[k]);
    if (coeff != 0.0) any_active = true;
    if (a.o_worst) a.o_worst[q * a.p + k] = dk;
  }
  const bool degenerate = !any_active && (a.m + a.p) > 0;
  if (a.o_value) a.o_value[q] = value;
  if (a.o_band) a.o_band[q] = band;
  if (a.o_flags)
    a.o_flags[q] = (uint8_t)(HJB_FILTER_OVERRIDE | (degenerate ? HJB_FILTER_DEGENERATE : 0) |
                             (ood ? HJB_FILTER_OOD : 0));
}

// interp_ex alone (grid.cpp:90-131), one thread per query
template <int ND>
__global__ void __launch_bounds__(128)
    k_interp(const __grid_constant__ DevGrid g, const double* __restrict__ f, long long nq,
             const double* __restrict__ x, double* value, uint8_t* ood_out, unsigned int* err) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= nq) return;
  uint32_t base[ND];
  double frac[ND];
  bool ood = false;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    const double xd = x[q * ND + d];
    if (!isfinite(xd)) {
      atomicOr(err, 1u);
      return;
    }
    double t = (xd - g.min[d]) / g.spacing[d];
    if (t < 0.0) {
      t = 0.0;
      ood = true;
    }
    const double tmax = (double)(g.n[d] - 1);
    if (t > tmax) {
      t = tmax;
      if (xd > g.max[d]) ood = true;
    }
    uint32_t i0 = (uint32_t)t;
    if (i0 > g.n[d] - 2) i0 = g.n[d] - 2;
    base[d] = i0;
    frac[d] = t - (double)i0;
  }
  double v = 0.0;
  for (int corner = 0; corner < (1 << ND); ++corner) {
    double w = 1.0;
    uint32_t lin = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      const bool hi = (corner >> d) & 1;
      w *= hi ? frac[d] : 1.0 - frac[d];
      lin += (base[d] + (hi ? 1u : 0u)) * g.stride[d];
    }
    if (w != 0.0) v += w * __ldg(f + lin);
  }
  if (value) value[q] = v;
  if (ood_out) ood_out[q] = ood ? 1 : 0;
}

template <int ND>
void launch_interp_nd(const DevGrid& g, const double* f, long long nq, const double* x,
                      double* value, uint8_t* ood, unsigned int* err, cudaStream_t s) {
  k_interp<ND><<<(unsigned)((nq + 127) / 128), 128, 0, s>>>(g, f, nq, x, value, ood, err);
}

// order-preserving unsigned key of a double (total order, -0 < +0)
__device__ __forceinline__ unsigned long long okey(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double unkey(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
#endif
}

__global__ void __launch_bounds__(256)
    k_reduce(const double* __restrict__ f, long long n, unsigned long long* keys) {
  unsigned long long mn = ~0ull, mx = 0ull;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = okey(__ldg(f + i));
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(keys, mn);
    atomicMax(keys + 1, mx);
  }
}

template <int ND>
void launch_nd(const FilterArgs& a, cudaStream_t s) {
  const unsigned blocks = (unsigned)((a.nq + 127) / 128);
  k_filter<ND><<<blocks, 128, 0, s>>>(a);
}

cudaError_t launch_filter(const FilterArgs& a, cudaStream_t s) {
  switch (a.g.nd) {
    case 1: launch_nd<1>(a, s); break;
    case 2: launch_nd<2>(a, s); break;
    case 3: launch_nd<3>(a, s); break;
    case 4: launch_nd<4>(a, s); break;
    case 5: launch_nd<5>(a, s); break;
    default: launch_nd<6>(a, s); break;
  }
  return cudaGetLastError();
}

// Validation shared by both entry points (SafetyFilter ctor, safety.cpp:76-84;
// make_context-style channel checks, solver.cpp:194-199).
int prepare_filter(const hjb_grid* gi, const hjb_model* mi, const hjb_dbounds* db,
                   const hjb_filter_config* cfg, int64_t nq, FilterArgs& a) {
  if (!gi || !mi || !db || !cfg) return set_err(HJB_ERR_INVALID_ARGUMENT, "filter: null argument");
  int rc;
  std::memset(&a, 0, sizeof a);
  if ((rc = make_grid(gi, a.g))) return rc;
  if (mi->state_dim != a.g.nd)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "SafetyFilter: grid rank does not match model");
  if (mi->control_dim < 0 || mi->control_dim > kMaxInput || mi->disturbance_dim < 0 ||
      mi->disturbance_dim > kMaxInput)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "model: bad dimensions");
  if (db->channels != mi->disturbance_dim)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "filter: disturbance channel count mismatch");
  if (cfg->mode != HJB_FILTER_OPTIMAL && cfg->mode != HJB_FILTER_FILTER)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "filter: unknown mode");
  if (nq < 0) return set_err(HJB_ERR_INVALID_ARGUMENT, "filter: negative query count");
  a.n = mi->state_dim;
  a.m = mi->control_dim;
  a.p = mi->disturbance_dim;
  for (int i = 0; i < a.n; ++i)
    for (int j = 0; j < kMaxInput; ++j) {
      a.B[i][j] = mi->control[i][j];
      a.C[i][j] = mi->disturbance[i][j];
    }
  for (int j = 0; j < a.m; ++j) {
    a.ulo[j] = mi->ubounds[j].lo;
    a.uhi[j] = mi->ubounds[j].hi;
  }
  a.per_node = db->per_node ? 1 : 0;
  for (int k = 0; k < a.p; ++k) {
    if (!db->per_node && !(db->constant[k].lo <= db->constant[k].hi))
      return set_err(HJB_ERR_INVALID_ARGUMENT, "IntervalField: lo > hi");
    a.dlo_c[k] = db->constant[k].lo;
    a.dhi_c[k] = db->constant[k].hi;
    a.dlo[k] = db->lo[k];
    a.dhi[k] = db->hi[k];
    if (db->per_node && (!db->lo[k] || !db->hi[k]))
      return set_err(HJB_ERR_INVALID_ARGUMENT, "dbounds: null field");
  }
  a.nq = nq;
  a.mode = cfg->mode;
  a.eta_floor = cfg->eta_floor;
  a.lambda = cfg->lambda;
  return HJB_OK;
}

int run_filter(hjb_context* ctx, FilterArgs& a) {
  CUDA_TRY(ctx->scratch.ensure(64));
  a.err = reinterpret_cast<unsigned int*>(ctx->scratch.p);
  CUDA_TRY(cudaMemsetAsync(a.err, 0, sizeof(unsigned int), ctx->stream));
  if (a.nq > 0) {
    CUDA_TRY(launch_filter(a, ctx->stream));
    ++ctx->launches;
  }
  unsigned int err = 0;
  CUDA_TRY(cudaMemcpyAsync(&err, a.err, sizeof err, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (err) return set_err(HJB_ERR_INVALID_ARGUMENT, "interp: non-finite query");
  return HJB_OK;
}

}  // namespace
}  // namespace hjb

using namespace hjb;

extern "C" {

int hjb_filter_batch_dev(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                         const hjb_dbounds* dbounds, const double* value, int64_t nq,
                         const double* x, const double* u_perf, const hjb_filter_config* cfg,
                         const hjb_filter_out* out) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  FilterArgs a;
  if ((rc = prepare_filter(grid, model, dbounds, cfg, nq, a))) return rc;
  if (nq > 0 && (!value || !x)) return set_err(HJB_ERR_INVALID_ARGUMENT, "filter: null field/query");
  if (nq > 0 && cfg->mode == HJB_FILTER_FILTER && a.m > 0 && !u_perf)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "filter: control dim mismatch");
  a.V = value;
  a.x = x;
  a.u_perf = u_perf;
  if (out) {
    a.o_value = out->value;
    a.o_band = out->band;
    a.o_control = out->control;
    a.o_worst = out->worst_disturbance;
    a.o_flags = out->flags;
  }
  return run_filter(ctx, a);
}

int hjb_filter_batch(hjb_context* ctx, const hjb_grid* grid, const hjb_model* model,
                     const hjb_dbounds* dbounds, const double* value, int64_t nq,
                     const double* x, const double* u_perf, const hjb_filter_config* cfg,
                     const hjb_filter_out* out) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  FilterArgs a;
  if ((rc = prepare_filter(grid, model, dbounds, cfg, nq, a))) return rc;
  if (nq > 0 && (!value || !x)) return set_err(HJB_ERR_INVALID_ARGUMENT, "filter: null field/query");
  if (nq > 0 && cfg->mode == HJB_FILTER_FILTER && a.m > 0 && !u_perf)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "filter: control dim mismatch");
  const size_t vb = static_cast<size_t>(a.g.size) * sizeof(double);
  const size_t nqs = static_cast<size_t>(nq);
  // one staging allocation: V | x | u_perf | value | band | control | worst | flags
  const size_t xb = nqs * a.n * sizeof(double), ub = nqs * a.m * sizeof(double);
  const size_t ob = nqs * sizeof(double), cb = nqs * a.m * sizeof(double),
               wb = nqs * a.p * sizeof(double), fb = (nqs + 7) / 8 * 8;
  CUDA_TRY(ctx->xbuf.ensure(vb + xb + ub + 2 * ob + cb + wb + fb));
  char* base = reinterpret_cast<char*>(ctx->xbuf.p);
  double* dV = reinterpret_cast<double*>(base);
  double* dx = reinterpret_cast<double*>(base + vb);
  double* du = reinterpret_cast<double*>(base + vb + xb);
  double* dval = reinterpret_cast<double*>(base + vb + xb + ub);
  double* dband = dval + nqs;
  double* dctl = dband + nqs;
  double* dworst = dctl + nqs * a.m;
  uint8_t* dflags = reinterpret_cast<uint8_t*>(dworst + nqs * a.p);
  CUDA_TRY(cudaMemcpyAsync(dV, value, vb, cudaMemcpyHostToDevice, ctx->stream));
  if (nq > 0) CUDA_TRY(cudaMemcpyAsync(dx, x, xb, cudaMemcpyHostToDevice, ctx->stream));
  if (nq > 0 && u_perf && ub)
    CUDA_TRY(cudaMemcpyAsync(du, u_perf, ub, cudaMemcpyHostToDevice, ctx->stream));
  hjb_dbounds dbs;
  if ((rc = stage_dbounds(ctx, dbounds, a.g.size, ctx->dbbuf, dbs))) return rc;
  for (int k = 0; k < a.p; ++k) {
    a.dlo[k] = dbs.lo[k];
    a.dhi[k] = dbs.hi[k];
  }
  a.V = dV;
  a.x = dx;
  a.u_perf = u_perf ? du : nullptr;
  a.o_value = dval;
  a.o_band = dband;
  a.o_control = dctl;
  a.o_worst = dworst;
  a.o_flags = dflags;
  if ((rc = run_filter(ctx, a))) return rc;
  if (out && nq > 0) {
    if (out->value) CUDA_TRY(cudaMemcpyAsync(out->value, dval, ob, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->band) CUDA_TRY(cudaMemcpyAsync(out->band, dband, ob, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->control && cb)
      CUDA_TRY(cudaMemcpyAsync(out->control, dctl, cb, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->worst_disturbance && wb)
      CUDA_TRY(cudaMemcpyAsync(out->worst_disturbance, dworst, wb, cudaMemcpyDeviceToHost,
                               ctx->stream));
    if (out->flags) CUDA_TRY(cudaMemcpyAsync(out->flags, dflags, nqs, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  }
  return HJB_OK;
}

int hjb_interp_batch_dev(hjb_context* ctx, const hjb_grid* grid, const double* field,
                         int64_t nq, const double* x, double* value, uint8_t* out_of_domain) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  DevGrid g;
  if ((rc = make_grid(grid, g))) return rc;
  if (nq < 0) return set_err(HJB_ERR_INVALID_ARGUMENT, "interp: negative query count");
  if (nq > 0 && (!field || !x)) return set_err(HJB_ERR_INVALID_ARGUMENT, "interp: null pointer");
  CUDA_TRY(ctx->scratch.ensure(64));
  unsigned int* err = reinterpret_cast<unsigned int*>(ctx->scratch.p);
  CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(unsigned int), ctx->stream));
  if (nq > 0) {
    switch (g.nd) {
      case 1: launch_interp_nd<1>(g, field, nq, x, value, out_of_domain, err, ctx->stream); break;
      case 2: launch_interp_nd<2>(g, field, nq, x, value, out_of_domain, err, ctx->stream); break;
      case 3: launch_interp_nd<3>(g, field, nq, x, value, out_of_domain, err, ctx->stream); break;
      case 4: launch_interp_nd<4>(g, field, nq, x, value, out_of_domain, err, ctx->stream); break;
      case 5: launch_interp_nd<5>(g, field, nq, x, value, out_of_domain, err, ctx->stream); break;
      default: launch_interp_nd<6>(g, field, nq, x, value, out_of_domain, err, ctx->stream); break;
    }
    CUDA_TRY(cudaGetLastError());
    ++ctx->launches;
  }
  unsigned int e = 0;
  CUDA_TRY(cudaMemcpyAsync(&e, err, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (e) return set_err(HJB_ERR_INVALID_ARGUMENT, "interp: non-finite query");
  return HJB_OK;
}

int hjb_field_reduce_dev(hjb_context* ctx, int64_t n, const double* field, double* min_out,
                         double* max_out) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  if (n <= 0 || !field) return set_err(HJB_ERR_INVALID_ARGUMENT, "reduce: empty field");
  CUDA_TRY(ctx->scratch.ensure(64));
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(ctx->scratch.p);
  const unsigned long long init[2] = {~0ull, 0ull};
  CUDA_TRY(cudaMemcpyAsync(keys, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
  const int sms = sm_count(ctx->device);
  const long long want = (n + 255) / 256;
  const unsigned blocks = (unsigned)std::min<long long>(want, 4LL * sms);
  k_reduce<<<blocks, 256, 0, ctx->stream>>>(field, n, keys);
  CUDA_TRY(cudaGetLastError());
  ++ctx->launches;
  unsigned long long out[2];
  CUDA_TRY(cudaMemcpyAsync(out, keys, sizeof out, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (min_out) *min_out = unkey(out[0]);
  if (max_out) *max_out = unkey(out[1]);
  return HJB_OK;
}

int hjb_malloc_dev(hjb_context* ctx, uint64_t bytes, void** out) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  if (!out) return set_err(HJB_ERR_INVALID_ARGUMENT, "malloc: null out");
  *out = nullptr;
  CUDA_TRY(cudaMalloc(out, bytes ? bytes : 1));
  return HJB_OK;
}

int hjb_free_dev(hjb_context* ctx, void* ptr) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (ptr) CUDA_TRY(cudaFree(ptr));
  return HJB_OK;
}

static int copy_sync(hjb_context* ctx, void* dst, const void* src, uint64_t bytes,
                     cudaMemcpyKind kind) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  if (bytes == 0) return HJB_OK;
  if (!dst || !src) return set_err(HJB_ERR_INVALID_ARGUMENT, "copy: null pointer");
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, kind, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return HJB_OK;
}

int hjb_copy_h2d(hjb_context* ctx, void* dst_dev, const void* src_host, uint64_t bytes) {
  return copy_sync(ctx, dst_dev, src_host, bytes, cudaMemcpyHostToDevice);
}
int hjb_copy_d2h(hjb_context* ctx, void* dst_host, const void* src_dev, uint64_t bytes) {
  return copy_sync(ctx, dst_host, src_dev, bytes, cudaMemcpyDeviceToHost);
}
int hjb_copy_d2d(hjb_context* ctx, void* dst_dev, const void* src_dev, uint64_t bytes) {
  return copy_sync(ctx, dst_dev, src_dev, bytes, cudaMemcpyDeviceToDevice);
}

}  // extern "C"
