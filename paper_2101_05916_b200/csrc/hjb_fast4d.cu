// hjb_fast4d.cu — the 4D Godunov sweep kernel, specialised for B200.
//
// Same arithmetic as the reference's update_chunk (solver.cpp:106-190,
// Godunov branch) on every node, organised for HBM streaming:
//
//  * internal padded layout [n0][n1][n2][n3p], n3p = n3 rounded up to even,
//    so every thread's 2-cell pencil along the contiguous axis is one aligned
//    16-byte vector (LDG.128 / STG.128);
//  * each thread owns one pencil at fixed (i1, i2) and MARCHES along axis 0
//    with a register queue V[i0-1], V[i0], V[i0+1], V[i0+2] (prefetch
//    distance 2), so every V element is streamed from HBM once per sweep;
//    the axis-0 face difference D+ of step i0 is reused as D- of step i0+1,
//    and the shared axis-3 face inside the pencil is computed once;
//  * in-plane neighbours (axes 1-3) come from L1/L2: CTAs cover T1 x T2
//    tiles of (i1, i2) rows and march in near-lockstep, so halo rows are
//    L2 hits;
//  * Godunov slopes of rows that do not depend on x0 are loop invariant and
//    live in registers for the whole march;
//  * the Godunov flux is evaluated in a branch-free, value-exact form: the
//    two products the reference forms (ha, hb) are computed identically and
//    the selection logic (solver.cpp:52-63) is restated with sign-bit tests
//    (every case where a sign test could differ from the reference's `> 0`
//    involves an exact zero operand, where both candidate results are +-0).
#include <cuda_runtime.h>

#include <cstdint>

#include "hjb_fast4d.cuh"

namespace hjb {

namespace {

__device__ __forceinline__ unsigned long long globaltimer_ns4() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool sign_clear(double x) { return __double2hiint(x) >= 0; }

// Godunov flux for a one-kink Hamiltonian (solver.cpp:44-63), value-exact.
__device__ __forceinline__ double flux(double pos, double neg, double dm, double dp) {
  const bool km = sign_clear(dm);  // dm "> 0" (+-0 classified by sign: see file header)
  const bool kp = sign_clear(dp);
  const double sm = km ? pos : neg;
  const double sp = kp ? pos : neg;
  const double ha = sm * dm;  // == reference kink_h(s, dminus)
  const double hb = sp * dp;  // == reference kink_h(s, dplus)
  const bool gt = ha > hb;
  double h;
  if (km == kp) {
    // same-signed gradients: the extremum over [dm,dp] of the linear piece is
    // attained at the upwind end: hb if the slope is >= 0, else ha
    h = sign_clear(sm) ? hb : ha;
  } else if (kp) {
    // dm <= 0 < dp: rarefaction, max(ha, hb) clamped at 0 from below
    h = gt ? ha : hb;
    h = sign_clear(h) ? h : 0.0;
  } else {
    // dp <= 0 < dm: shock, min(ha, hb) clamped at 0 from above
    h = gt ? hb : ha;
    h = sign_clear(h) ? 0.0 : h;
  }
  return h;
}

struct ShapePlanar {  // NearHoverPlanar4D rows: x1 | tan(x2) | x2 + x3 | x2
  __host__ __device__ static constexpr int A(int d) { return d == 0 ? 1 : 2; }
  __host__ __device__ static constexpr int B(int d) { return d == 2 ? 3 : -1; }
};
struct ShapeTwin {  // TwinDoubleIntegrator rows: x1 | const | x3 | const
  __host__ __device__ static constexpr int A(int d) { return d == 0 ? 1 : d == 2 ? 3 : -1; }
  __host__ __device__ static constexpr int B(int) { return -1; }
};

template <class S>
__device__ __forceinline__ uint32_t pick(int axis, uint32_t i1, uint32_t i2, uint32_t i3) {
  return axis == 1 ? i1 : axis == 2 ? i2 : axis == 3 ? i3 : 0u;
}

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

__device__ __forceinline__ double2 ldg2_stream(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned long long umax64(unsigned long long a,
                                                     unsigned long long b) {
  return a > b ? a : b;
}

template <class S>
__global__ void __launch_bounds__(512, 1) k_fast4d(const __grid_constant__ Fast4dArgs a) {
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
  const uint32_t n0 = a.n[0], n1 = a.n[1], n2 = a.n[2], n3 = a.n[3];
  const uint32_t n3p = a.n3p;
  const uint32_t J = n3p >> 1;

  // block -> (tile_i1, tile_i2, i0 chunk)
  uint32_t b = blockIdx.x;
  const uint32_t chunk = b % a.nchunks;
  b /= a.nchunks;
  const uint32_t t2 = b % a.tiles2;
  const uint32_t t1 = b / a.tiles2;
  const uint32_t t = threadIdx.x;
  const uint32_t r = t / J;
  const uint32_t j = t - r * J;
  const uint32_t r1 = r / a.T2;
  const uint32_t r2 = r - r1 * a.T2;
  const uint32_t i1 = t1 * a.T1 + r1;
  const uint32_t i2 = t2 * a.T2 + r2;
  const bool active = r < a.T1 * a.T2 && i1 < n1 && i2 < n2;
  unsigned long long mbits = 0ull;

  if (active) {
    const uint32_t i3 = 2 * j;
    const bool has1 = i3 + 1 < n3;          // second pencil cell is real
    const bool has_r = i3 + 2 < n3;         // right neighbour exists
    const bool has_l = i3 > 0;
    const bool m1 = i1 > 0, p1 = i1 + 1 < n1;
    const bool m2 = i2 > 0, p2 = i2 + 1 < n2;
    const uint64_t s2 = n3p;
    const uint64_t s1 = static_cast<uint64_t>(n2) * n3p;
    const uint64_t s0 = static_cast<uint64_t>(n1) * s1;
    const double inv0 = a.inv[0], inv1 = a.inv[1], inv2 = a.inv[2], inv3 = a.inv[3];

    // loop-invariant Godunov slopes (rows never depend on x0 in this path)
    double pos[4][2], neg[4][2];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t ka = pick<S>(S::A(d), i1, i2, i3 + c);
        if (S::B(d) < 0) {
          pos[d][c] = __ldg(a.tab + a.off_pos[d] + ka);
          neg[d][c] = __ldg(a.tab + a.off_neg[d] + ka);
        } else {
          const uint32_t kb = pick<S>(S::B(d), i1, i2, i3 + c);
          const double dr = __ldg(a.tab + a.off_a[d] + ka) + __ldg(a.tab + a.off_b[d] + kb);
          pos[d][c] = dr;
          neg[d][c] = dr;
        }
      }
    }

    const uint32_t c0 = chunk * a.L;
    const uint32_t c1 = min(c0 + a.L, n0);
    const uint64_t rowoff = (static_cast<uint64_t>(i1) * n2 + i2) * n3p + i3;
    const double* vp = src + rowoff;  // pencil at plane 0
    double* op = dst + rowoff;
    const double* cp = a.c + rowoff;

    double2 vprev = make_double2(0.0, 0.0);
    double2 vcur = ldg2(vp + c0 * s0);
    double2 vnext = make_double2(0.0, 0.0);
    double2 vnn = make_double2(0.0, 0.0);
    if (c0 > 0) vprev = ldg2(vp + (c0 - 1) * s0);
    if (c0 + 1 < n0) vnext = ldg2(vp + (c0 + 1) * s0);
    double2 ccur = ldg2_stream(cp + c0 * s0);
    // axis-0 D- of the first step
    double dm0a = 0.0, dm0b = 0.0;
    if (c0 > 0) {
      dm0a = (vcur.x - vprev.x) * inv0;
      dm0b = (vcur.y - vprev.y) * inv0;
    }
    for (uint32_t i0 = c0; i0 < c1; ++i0) {
      const uint64_t pl = static_cast<uint64_t>(i0) * s0;
      // prefetch V[i0+2] and c[i0+1]
      if (i0 + 2 < n0) vnn = ldg2(vp + pl + 2 * s0);
      double2 cnext = make_double2(0.0, 0.0);
      if (i0 + 1 < c1) cnext = ldg2_stream(cp + pl + s0);
      // in-plane neighbours at plane i0
      const double* q = vp + pl;
      double2 a1m = m1 ? ldg2(q - s1) : vcur;
      double2 a1p = p1 ? ldg2(q + s1) : vcur;
      double2 a2m = m2 ? ldg2(q - s2) : vcur;
      double2 a2p = p2 ? ldg2(q + s2) : vcur;
      const double vl = has_l ? __ldg(q - 1) : 0.0;
      const double vr = has_r ? __ldg(q + 2) : 0.0;

      // axis 0: D+ (shared with the next step's D-)
      double dp0a = 0.0, dp0b = 0.0;
      if (i0 + 1 < n0) {
        dp0a = (vnext.x - vcur.x) * inv0;
        dp0b = (vnext.y - vcur.y) * inv0;
      }
      // axis 1
      const double dm1a = m1 ? (vcur.x - a1m.x) * inv1 : 0.0;
      const double dm1b = m1 ? (vcur.y - a1m.y) * inv1 : 0.0;
      const double dp1a = p1 ? (a1p.x - vcur.x) * inv1 : 0.0;
      const double dp1b = p1 ? (a1p.y - vcur.y) * inv1 : 0.0;
      // axis 2
      const double dm2a = m2 ? (vcur.x - a2m.x) * inv2 : 0.0;
      const double dm2b = m2 ? (vcur.y - a2m.y) * inv2 : 0.0;
      const double dp2a = p2 ? (a2p.x - vcur.x) * inv2 : 0.0;
      const double dp2b = p2 ? (a2p.y - vcur.y) * inv2 : 0.0;
      // axis 3: faces (l|x), (x|y), (y|r)
      const double f3m = has_l ? (vcur.x - vl) * inv3 : 0.0;
      const double f3c = has1 ? (vcur.y - vcur.x) * inv3 : 0.0;
      const double f3p = has_r ? (vr - vcur.y) * inv3 : 0.0;

      // Hhat = sum_d flux_d, in d order (hhat starts at 0.0: 0.0 + h0 == h0 in value)
      double ha_ = flux(pos[0][0], neg[0][0], dm0a, dp0a);
      ha_ += flux(pos[1][0], neg[1][0], dm1a, dp1a);
      ha_ += flux(pos[2][0], neg[2][0], dm2a, dp2a);
      ha_ += flux(pos[3][0], neg[3][0], f3m, f3c);
      double hb_ = flux(pos[0][1], neg[0][1], dm0b, dp0b);
      hb_ += flux(pos[1][1], neg[1][1], dm1b, dp1b);
      hb_ += flux(pos[2][1], neg[2][1], dm2b, dp2b);
      hb_ += flux(pos[3][1], neg[3][1], f3c, f3p);

      const double sa = vcur.x + a.dt * ha_;
      const double sb = vcur.y + a.dt * hb_;
      double2 o;
      o.x = sa > ccur.x ? sa : ccur.x;
      o.y = sb > ccur.y ? sb : ccur.y;
      *reinterpret_cast<double2*>(op + pl) = o;
      const double dva = fabs(o.x - vcur.x);
      const double dvb = fabs(o.y - vcur.y);
      // NaN never wins (reference: `if (dv > max_dv)`); its bit pattern would
      // order above +inf, so it is filtered explicitly
      const unsigned long long ba =
          dva == dva ? (unsigned long long)__double_as_longlong(dva) : 0ull;
      unsigned long long bb =
          dvb == dvb ? (unsigned long long)__double_as_longlong(dvb) : 0ull;
      if (!has1) bb = 0ull;
      mbits = umax64(mbits, umax64(ba, bb));

      // rotate the queue
      dm0a = dp0a;
      dm0b = dp0b;
      vprev = vcur;
      vcur = vnext;
      vnext = vnn;
      ccur = cnext;
    }
    (void)vprev;
  }

  // CTA max -> global, last CTA runs the sweep epilogue (solver.cpp:347-369)
  __shared__ unsigned long long part[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mbits = umax64(mbits, __shfl_xor_sync(0xffffffffu, mbits, o));
  if (lane == 0) part[warp] = mbits;
  __syncthreads();
  if (warp != 0) return;
  mbits = lane < (int)(blockDim.x >> 5) ? part[lane] : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mbits = umax64(mbits, __shfl_xor_sync(0xffffffffu, mbits, o));
  if (lane != 0) return;
  LoopState* st = a.st;
  if (mbits) atomicMax(&st->maxdv_bits, mbits);
  if (!a.loop) return;
  __threadfence();
  const unsigned int ticket = atomicAdd(&st->blocks_done, 1u);
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  const double max_dv = __longlong_as_double(atomicAdd(&st->maxdv_bits, 0ull));
  const double residual = max_dv / st->dt;
  const long long iter = st->iter + 1;
  st->iter = iter;
  if (iter - 1 < st->history_cap) {
    if (st->history) st->history[iter - 1] = residual;
    if (st->wall_history)
      st->wall_history[iter - 1] = (double)(globaltimer_ns4() - st->t0_ns) * 1e-6;
  }
  st->last_residual = residual;
  bool stop = false;
  if (residual < st->tol) {
    st->converged = 1;
    stop = true;
  } else {
    if (iter == 1) st->first_residual = residual;
    const double mr0 = st->min_residual;
    const double mr = residual < mr0 ? residual : mr0;
    st->min_residual = mr;
    const double first = st->first_residual;
    const double base = mr < first ? first : mr;
    if (!isfinite(residual) || residual > 10.0 * base) {
      st->status = HJB_ERR_DIVERGED;
      stop = true;
    }
  }
  if (iter >= st->max_iters) stop = true;
  if (st->horizon > 0.0 && (double)iter * st->dt >= st->horizon) stop = true;
  st->maxdv_bits = 0ull;
  st->blocks_done = 0u;
  if (stop) {
    st->done = 1;
    if (a.use_handle) cudaGraphSetConditional(a.handle, 0u);
  }
  __threadfence();
}

// padded <-> reference layout
__global__ void k_pad4(const double* __restrict__ in, double* __restrict__ out, uint64_t rows,
                       uint32_t n3, uint32_t n3p, double fill) {
  const uint64_t total = rows * n3p;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = i / n3p;
    const uint32_t k = static_cast<uint32_t>(i - row * n3p);
    out[i] = k < n3 ? in[row * n3 + k] : fill;
  }
}

__global__ void k_unpad4(const double* __restrict__ in, double* __restrict__ out, uint64_t rows,
                         uint32_t n3, uint32_t n3p) {
  const uint64_t total = rows * n3;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = i / n3;
    const uint32_t k = static_cast<uint32_t>(i - row * n3);
    out[i] = in[row * n3p + k];
  }
}

}  // namespace

int fast4d_shape(const DevGrid& g, const DevModel& m, int scheme) {
  if (g.nd != 4 || scheme != 0 || m.per_node) return -1;
  if ((g.n[3] + 1) / 2 > 512) return -1;
  int A[4], B[4];
  for (int d = 0; d < 4; ++d) {
    const DevRow& r = m.row[d];
    if (r.folded) {
      A[d] = r.axis_a;
      B[d] = -1;
    } else if (r.axis_b >= 0 && r.n_uadd == 0 && r.n_dterm == 0 && !r.constant_drift) {
      A[d] = r.axis_a;
      B[d] = r.axis_b;
    } else {
      return -1;
    }
    if (A[d] == 0 || B[d] == 0) return -1;
  }
  auto match = [&](const int* a, const int* b) {
    for (int d = 0; d < 4; ++d)
      if (a[d] != A[d] || b[d] != B[d]) return false;
    return true;
  };
  static const int pa[4] = {1, 2, 2, 2}, pb[4] = {-1, -1, 3, -1};
  static const int ta[4] = {1, -1, 3, -1}, tb[4] = {-1, -1, -1, -1};
  if (match(pa, pb)) return 0;
  if (match(ta, tb)) return 1;
  return -1;
}

void fast4d_config(const DevGrid& g, int sms, Fast4dArgs& a) {
  for (int d = 0; d < 4; ++d) {
    a.n[d] = g.n[d];
    a.inv[d] = g.inv_spacing[d];
  }
  a.n3p = g.n[3] + (g.n[3] & 1u);
  const uint32_t J = a.n3p / 2;
  // rows per CTA so that a CTA has ~256-512 threads
  uint32_t R = 512 / J;
  if (R < 1) R = 1;
  uint32_t T2 = 1;
  while (T2 * T2 < R) ++T2;
  if (T2 > g.n[2]) T2 = g.n[2];
  uint32_t T1 = R / T2;
  if (T1 < 1) T1 = 1;
  if (T1 > g.n[1]) T1 = g.n[1];
  a.T1 = T1;
  a.T2 = T2;
  a.tiles1 = (g.n[1] + T1 - 1) / T1;
  a.tiles2 = (g.n[2] + T2 - 1) / T2;
  a.threads = ((T1 * T2 * J + 31) / 32) * 32;
  const uint32_t tiles = a.tiles1 * a.tiles2;
  const uint32_t want = static_cast<uint32_t>(sms) * 4;  // ~2 CTAs/SM x 2 waves
  uint32_t nch = (want + tiles - 1) / tiles;
  if (nch < 1) nch = 1;
  uint32_t L = (g.n[0] + nch - 1) / nch;
  if (L < 4) L = 4;
  a.L = L;
  a.nchunks = (g.n[0] + L - 1) / L;
  a.blocks = tiles * a.nchunks;
}

cudaError_t launch_fast4d(const Fast4dArgs& a, int shape, cudaStream_t s) {
  if (shape == 0)
    k_fast4d<ShapePlanar><<<a.blocks, a.threads, 0, s>>>(a);
  else
    k_fast4d<ShapeTwin><<<a.blocks, a.threads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pad4(const double* in, double* out, uint64_t rows, uint32_t n3, uint32_t n3p,
                        cudaStream_t s) {
  k_pad4<<<148 * 8, 256, 0, s>>>(in, out, rows, n3, n3p, 0.0);
  return cudaGetLastError();
}

cudaError_t launch_unpad4(const double* in, double* out, uint64_t rows, uint32_t n3,
                          uint32_t n3p, cudaStream_t s) {
  k_unpad4<<<148 * 8, 256, 0, s>>>(in, out, rows, n3, n3p);
  return cudaGetLastError();
}

}  // namespace hjb
