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
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include <cudaTypedefs.h>

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

// ---- mbarrier / bulk-copy primitives (PTX ISA 8.x, sm_90+; TMA engine) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 4D TMA tile load (tensor map in kernel-parameter space), OOB -> zeros
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, int c0, int c1,
                                          int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ double2 lds2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}

// One CTA = a T1 x T2 tile of (i1, i2) rows (full contiguous rows of n3p),
// marching i0 over [c0, c1).  One elected thread streams each V plane
// (tile + 1-row halo in i1 and i2, out-of-range rows zero-filled by the TMA
// unit) and each c plane (tile) into shared-memory rings with a single 4D
// tensor copy each; full/empty mbarriers pipeline the planes, so no
// block-wide barrier is needed inside the march.  Every thread owns one
// 2-cell pencil.
template <class S>
__global__ void __launch_bounds__(448, 2) k_fast4d(const __grid_constant__ Fast4dArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const double* src;
  double* dst;
  const CUtensorMap* vmap;
  if (a.loop) {
    if (*(volatile int*)&a.st->done) return;
    const long long it = a.st->iter;
    src = (it & 1) ? a.buf1 : a.buf0;
    dst = (it & 1) ? a.buf0 : a.buf1;
    vmap = (it & 1) ? &a.map1 : &a.map0;
  } else {
    src = a.src;
    dst = a.dst;
    vmap = &a.map0;
  }
  (void)src;
  const uint32_t n0 = a.n[0], n1 = a.n[1], n2 = a.n[2], n3 = a.n[3];
  const uint32_t n3p = a.n3p;
  const uint32_t J = n3p >> 1;
  const uint32_t T1 = a.T1, T2 = a.T2;
  const uint32_t W2 = T2 + 2;
  const uint32_t RC = T1 * T2;        // c rows per slot
  constexpr uint32_t SV = 4;          // V ring
  constexpr uint32_t SC = 2;          // c ring
  double* vring = reinterpret_cast<double*>(smem_raw);
  double* cring = reinterpret_cast<double*>(smem_raw + SV * a.vslot_bytes);
  uint64_t* full_v = reinterpret_cast<uint64_t*>(smem_raw + SV * a.vslot_bytes + SC * a.cslot_bytes);
  uint64_t* empty_v = full_v + SV;
  uint64_t* full_c = empty_v + SV;
  uint64_t* empty_c = full_c + SC;
  const uint32_t vslot = a.vslot_bytes / 8, cslot = a.cslot_bytes / 8;  // in doubles

  uint32_t b = blockIdx.x;
  const uint32_t chunk = b % a.nchunks;
  b /= a.nchunks;
  const uint32_t t2 = b % a.tiles2;
  const uint32_t t1 = b / a.tiles2;
  const uint32_t base1 = t1 * T1, base2 = t2 * T2;
  const uint32_t c0 = chunk * a.L;
  const uint32_t c1 = min(c0 + a.L, n0);
  const uint64_t s2 = n3p;
  const uint64_t s1 = static_cast<uint64_t>(n2) * n3p;
  const uint64_t s0 = static_cast<uint64_t>(n1) * s1;
  const uint32_t nwarps = blockDim.x >> 5;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = threadIdx.x == 0;

  if (producer) {
    for (uint32_t k = 0; k < SV; ++k) {
      mbar_init(full_v + k, 1);
      mbar_init(empty_v + k, nwarps);
    }
    for (uint32_t k = 0; k < SC; ++k) {
      mbar_init(full_c + k, 1);
      mbar_init(empty_c + k, nwarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // producer state (thread 0 only): per-slot parity bits of the empty barriers
  uint32_t pv = 0, pc = 0;
  const uint32_t last_v = (c1 < n0) ? c1 : n0 - 1;  // last V plane this chunk reads
  auto issue_v = [&](uint32_t p) {
    const uint32_t sl = p % SV;
    mbar_wait(empty_v + sl, ((pv >> sl) & 1u) ^ 1u);
    pv ^= 1u << sl;
    mbar_arrive_expect_tx(full_v + sl, a.vbox_bytes);
    tma_load4(vring + sl * vslot, vmap, 0, (int)base2 - 1, (int)base1 - 1, (int)p, full_v + sl);
  };
  auto issue_c = [&](uint32_t p) {
    const uint32_t sl = p % SC;
    mbar_wait(empty_c + sl, ((pc >> sl) & 1u) ^ 1u);
    pc ^= 1u << sl;
    mbar_arrive_expect_tx(full_c + sl, a.cbox_bytes);
    tma_load4(cring + sl * cslot, &a.mapc, 0, (int)base2, (int)base1, (int)p, full_c + sl);
  };

  const uint32_t pfirst = c0 > 0 ? c0 - 1 : 0;
  if (producer) {
    for (uint32_t p = pfirst; p <= c0 + 1 && p <= last_v; ++p) issue_v(p);
    issue_c(c0);
  }
  uint32_t fv = 0, fc = 0;  // consumer parity bits of the full barriers

  const uint32_t t = threadIdx.x;
  const uint32_t r = t / J;
  const uint32_t j = t - r * J;
  const uint32_t r1 = r / T2;
  const uint32_t r2 = r - r1 * T2;
  const uint32_t i1 = base1 + r1;
  const uint32_t i2 = base2 + r2;
  const bool active = r < RC && i1 < n1 && i2 < n2;
  const uint32_t i3 = 2 * j;
  const bool has1 = i3 + 1 < n3;
  const bool has_r = i3 + 2 < n3;
  const bool has_l = i3 > 0;
  const bool m1 = i1 > 0, p1 = i1 + 1 < n1;
  const bool m2 = i2 > 0, p2 = i2 + 1 < n2;
  const double inv0 = a.inv[0], inv1 = a.inv[1], inv2 = a.inv[2], inv3 = a.inv[3];
  const uint32_t own = ((r1 + 1) * W2 + (r2 + 1)) * n3p + i3;  // pencil offset in a V slot
  const uint32_t cown = r * n3p + i3;                          // pencil offset in a c slot
  double* op = dst + static_cast<uint64_t>(i1) * s1 + static_cast<uint64_t>(i2) * s2 + i3;

  double pos[4][2], neg[4][2];
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    // rows that do not depend on x3 hold one slope pair for the whole pencil
    constexpr int dummy = 0;
    (void)dummy;
    const bool per_cell = S::A(d) == 3 || S::B(d) == 3;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (c == 1 && !per_cell) {
        pos[d][1] = pos[d][0];
        neg[d][1] = neg[d][0];
        continue;
      }
      const uint32_t ka = active ? pick<S>(S::A(d), i1, i2, min(i3 + c, n3 - 1)) : 0u;
      if (S::B(d) < 0) {
        pos[d][c] = __ldg(a.tab + a.off_pos[d] + ka);
        neg[d][c] = __ldg(a.tab + a.off_neg[d] + ka);
      } else {
        const uint32_t kb = active ? pick<S>(S::B(d), i1, i2, min(i3 + c, n3 - 1)) : 0u;
        const double dr = __ldg(a.tab + a.off_a[d] + ka) + __ldg(a.tab + a.off_b[d] + kb);
        pos[d][c] = dr;
        neg[d][c] = dr;
      }
    }
  }

  auto wait_v = [&](uint32_t p) {
    const uint32_t sl = p % SV;
    mbar_wait(full_v + sl, (fv >> sl) & 1u);
    fv ^= 1u << sl;
  };
  auto release_v = [&](uint32_t p) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_v + (p % SV));
  };

  // prologue planes c0-1, c0
  for (uint32_t p = pfirst; p <= c0; ++p) wait_v(p);
  double2 vprev = make_double2(0.0, 0.0), vcur = make_double2(0.0, 0.0);
  if (active) {
    if (c0 > 0) vprev = lds2(vring + ((c0 - 1) % SV) * vslot + own);
    vcur = lds2(vring + (c0 % SV) * vslot + own);
  }
  if (c0 > 0) release_v(c0 - 1);
  double dm0a = 0.0, dm0b = 0.0;
  if (c0 > 0) {
    dm0a = (vcur.x - vprev.x) * inv0;
    dm0b = (vcur.y - vprev.y) * inv0;
  }
  unsigned long long mbits = 0ull;

  for (uint32_t i0 = c0; i0 < c1; ++i0) {
    if (producer) {
      if (i0 + 2 <= last_v) issue_v(i0 + 2);
      if (i0 + 1 < c1) issue_c(i0 + 1);
    }
    if (i0 + 1 < n0) wait_v(i0 + 1);
    {
      const uint32_t sl = i0 % SC;
      mbar_wait(full_c + sl, (fc >> sl) & 1u);
      fc ^= 1u << sl;
    }
    if (active) {
      const double* cur = vring + (i0 % SV) * vslot + own;
      double2 vnext = vcur;
      if (i0 + 1 < n0) vnext = lds2(vring + ((i0 + 1) % SV) * vslot + own);
      const double2 cc = lds2(cring + (i0 % SC) * cslot + cown);
      const double2 a1m = lds2(cur - W2 * n3p);
      const double2 a1p = lds2(cur + W2 * n3p);
      const double2 a2m = lds2(cur - n3p);
      const double2 a2p = lds2(cur + n3p);
      const double vl = has_l ? cur[-1] : 0.0;
      const double vr = has_r ? cur[2] : 0.0;

      double dp0a = 0.0, dp0b = 0.0;
      if (i0 + 1 < n0) {
        dp0a = (vnext.x - vcur.x) * inv0;
        dp0b = (vnext.y - vcur.y) * inv0;
      }
      const double dm1a = m1 ? (vcur.x - a1m.x) * inv1 : 0.0;
      const double dm1b = m1 ? (vcur.y - a1m.y) * inv1 : 0.0;
      const double dp1a = p1 ? (a1p.x - vcur.x) * inv1 : 0.0;
      const double dp1b = p1 ? (a1p.y - vcur.y) * inv1 : 0.0;
      const double dm2a = m2 ? (vcur.x - a2m.x) * inv2 : 0.0;
      const double dm2b = m2 ? (vcur.y - a2m.y) * inv2 : 0.0;
      const double dp2a = p2 ? (a2p.x - vcur.x) * inv2 : 0.0;
      const double dp2b = p2 ? (a2p.y - vcur.y) * inv2 : 0.0;
      const double f3m = has_l ? (vcur.x - vl) * inv3 : 0.0;
      const double f3c = has1 ? (vcur.y - vcur.x) * inv3 : 0.0;
      const double f3p = has_r ? (vr - vcur.y) * inv3 : 0.0;

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
      o.x = sa > cc.x ? sa : cc.x;
      o.y = sb > cc.y ? sb : cc.y;
      *reinterpret_cast<double2*>(op + static_cast<uint64_t>(i0) * s0) = o;
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

      dm0a = dp0a;
      dm0b = dp0b;
      vprev = vcur;
      vcur = vnext;
    }
    // plane i0 (V) and c plane i0 are no longer read by this warp
    release_v(i0);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_c + (i0 % SC));
  }
  (void)vprev;

  // CTA max -> global, last CTA runs the sweep epilogue (solver.cpp:347-369)
  __shared__ unsigned long long part[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mbits = umax64(mbits, __shfl_xor_sync(0xffffffffu, mbits, o));
  if (lane == 0) part[warp] = mbits;
  __syncthreads();
  if (warp != 0) return;
  mbits = lane < (blockDim.x >> 5) ? part[lane] : 0ull;
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
  if (g.n[3] + (g.n[3] & 1u) > 256) return -1;  // TMA box extent limit
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

static uint32_t round128(size_t b) { return static_cast<uint32_t>((b + 127) / 128 * 128); }

static size_t fast4d_smem(uint32_t T1, uint32_t T2, uint32_t n3p) {
  const size_t rv = (T1 + 2) * (T2 + 2), rc = T1 * T2;
  return 4 * (size_t)round128(rv * n3p * sizeof(double)) +
         2 * (size_t)round128(rc * n3p * sizeof(double)) + 12 * sizeof(uint64_t);
}

void fast4d_config(const DevGrid& g, int sms, Fast4dArgs& a) {
  for (int d = 0; d < 4; ++d) {
    a.n[d] = g.n[d];
    a.inv[d] = g.inv_spacing[d];
  }
  a.n3p = g.n[3] + (g.n[3] & 1u);
  const uint32_t J = a.n3p / 2;
  // rows per CTA: <= 448 threads, shared-memory rings small enough for 2 CTAs/SM
  uint32_t R = 448 / J;
  if (R < 1) R = 1;
  uint32_t T1 = 1, T2 = 1;
  for (;;) {
    T2 = 1;
    while (T2 * T2 < R) ++T2;
    if (T2 > g.n[2]) T2 = g.n[2];
    T1 = R / T2;
    if (T1 < 1) T1 = 1;
    if (T1 > g.n[1]) T1 = g.n[1];
    if (fast4d_smem(T1, T2, a.n3p) <= 110 * 1024 || R == 1) break;
    --R;
  }
  a.T1 = T1;
  a.T2 = T2;
  a.tiles1 = (g.n[1] + T1 - 1) / T1;
  a.tiles2 = (g.n[2] + T2 - 1) / T2;
  a.threads = ((T1 * T2 * J + 31) / 32) * 32;
  a.smem = static_cast<uint32_t>(fast4d_smem(T1, T2, a.n3p));
  a.vbox_bytes = (T1 + 2) * (T2 + 2) * a.n3p * 8u;
  a.cbox_bytes = T1 * T2 * a.n3p * 8u;
  a.vslot_bytes = round128(a.vbox_bytes);
  a.cslot_bytes = round128(a.cbox_bytes);
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
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_fast4d<ShapePlanar>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(k_fast4d<ShapeTwin>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_set = true;
  }
  if (shape == 0)
    k_fast4d<ShapePlanar><<<a.blocks, a.threads, a.smem, s>>>(a);
  else
    k_fast4d<ShapeTwin><<<a.blocks, a.threads, a.smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t fast4d_make_maps(Fast4dArgs& a, double* buf0, double* buf1, const double* c) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[4] = {a.n3p, a.n[2], a.n[1], a.n[0]};
  const cuuint64_t strides[3] = {(cuuint64_t)a.n3p * 8, (cuuint64_t)a.n3p * a.n[2] * 8,
                                 (cuuint64_t)a.n3p * a.n[2] * a.n[1] * 8};
  const cuuint32_t vbox[4] = {a.n3p, a.T2 + 2, a.T1 + 2, 1};
  const cuuint32_t cbox[4] = {a.n3p, a.T2, a.T1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMap* maps[3] = {&a.map0, &a.map1, &a.mapc};
  const void* ptrs[3] = {buf0, buf1, c};
  for (int k = 0; k < 3; ++k) {
    CUresult r = encode(maps[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(ptrs[k]),
                        dims, strides, k < 2 ? vbox : cbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  return cudaSuccess;
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
