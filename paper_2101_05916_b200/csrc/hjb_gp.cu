// GP disturbance bounds on the solver grid: the step before
// the path.  Reference: bounds_on_grid (proj/src/gp.cpp:211-249) evaluates
// GpModel::predict (gp.cpp:188-208) at EVERY grid node — n_train kernel
// values, a dot product and an O(n_train^2) forward substitution per node,
// although the prediction depends only on the node's coordinates along the
// channel's input dims (sim.cpp:605,647,660 condition on axis 0 only).
//
// B200 design:
//  * the distinct GP inputs are enumerated once per channel: M = prod of the
//    grid extents over input_dims (51 for a 51^4 grid conditioned on x);
//  * k*(x_m, x_i) = signal_var * exp(-0.5 q) is tabulated on the host with
//    the reference's own arithmetic (gp.cpp:22-30; glibc exp, the one
//    transcendental of the path, like the tan tables of the drift);
//  * k_gp_posterior: one CTA per distinct input.  mean = sum k*_i alpha_i and
//    the forward substitution v = L^-1 k* keep the reference's operation order
//    bit for bit: for row i, s = k*_i; s -= L[i][j] v_j for j = 0..i-1; v_i =
//    s / L[i][i].  Rows are spread over the threads; step j is one barrier:
//    the owner of row j finalises v_j, every row i > j subtracts its term,
//    which is exactly the reference's j order per row.  L is read column-
//    major (coalesced across rows) with a register prefetch 8 steps ahead;
//  * k_gp_broadcast: lo/hi of every node = the table entry of its input
//    point, 16 B per node per channel written once — HBM-bound.
// Results are bitwise those of the CPU restatement (oracle/hj_oracle.c,
// hjo_gp_bounds_on_grid) which follows gp.cpp line by line.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hjb_internal.cuh"

namespace hjb {
namespace {

// register prefetch depth of the L columns (R rows per thread)
template <int R>
struct Pf {
  static constexpr int D = R >= 8 ? 1 : 8 / R;
};

// One CTA per query point p.  w (shared) holds the running s_i of every row,
// finalised in place into v_i.  R = rows per thread (row i -> thread i % T).
template <int R>
__global__ void __launch_bounds__(1024) k_gp_posterior(
    const double* __restrict__ kstar, int n, const double* __restrict__ alpha,
    const double* __restrict__ lt, int ldt, const double* __restrict__ diag, double signal_var,
    double noise_var, double confidence, double* __restrict__ out_a,
    double* __restrict__ out_b, int bounds) {
  extern __shared__ double w[];
  const int T = blockDim.x, t = threadIdx.x;
  const double* ks = kstar + static_cast<size_t>(blockIdx.x) * n;
  for (int i = t; i < n; i += T) w[i] = ks[i];
  __syncthreads();
  // running sums of this thread's rows in registers
  double s[R];
#pragma unroll
  for (int r = 0; r < R; ++r) s[r] = (t + r * T < n) ? w[t + r * T] : 0.0;
  constexpr int kPrefetch = Pf<R>::D;
  double cur[kPrefetch][R], nxt[kPrefetch][R];
  auto load = [&](int j0, double (&buf)[kPrefetch][R]) {
#pragma unroll
    for (int u = 0; u < kPrefetch; ++u) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = t + r * T, j = j0 + u;
        buf[u][r] = (j < n && i > j && i < n) ? __ldg(lt + static_cast<size_t>(j) * ldt + i) : 0.0;
      }
    }
  };
  load(0, cur);
  for (int j0 = 0; j0 < n; j0 += kPrefetch) {
    load(j0 + kPrefetch, nxt);
#pragma unroll
    for (int u = 0; u < kPrefetch; ++u) {
      const int j = j0 + u;
      if (j >= n) break;  // uniform across the CTA
      // the owner of row j finalises v_j = s_j / L[j][j] (gp.cpp:201)
      if (j % T == t) {
        const int r = j / T;
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (q == r) {
            s[q] = s[q] / diag[j];
            w[j] = s[q];
          }
      }
      __syncthreads();
      const double vj = w[j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = t + r * T;
        if (i > j && i < n) s[r] = s[r] - cur[u][r] * vj;  // gp.cpp:200
      }
    }
#pragma unroll
    for (int u = 0; u < kPrefetch; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) cur[u][r] = nxt[u][r];
  }
  __syncthreads();
  if (t == 0) {
    double mean = 0.0;  // gp.cpp:193-194
    for (int i = 0; i < n; ++i) mean += ks[i] * alpha[i];
    double var = signal_var;  // gp.cpp:204-205
    for (int i = 0; i < n; ++i) var -= w[i] * w[i];
    var = var < 0.0 ? 0.0 : var;  // std::max(var, 0.0)
    if (bounds) {  // gp.cpp:241-245
      const double band = confidence * sqrt(var + noise_var);
      out_a[blockIdx.x] = mean - band;
      out_b[blockIdx.x] = mean + band;
    } else {
      out_a[blockIdx.x] = mean;
      out_b[blockIdx.x] = var;
    }
  }
}

// ---- mbarrier / 1D bulk copy (TMA engine) ----
__device__ __forceinline__ uint32_t gp_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void gp_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "GPWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra GPWAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gp_column(uint32_t dst, const double* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

// Correctly rounded s / d from y = RN(1/d) (Markstein: q = RN(s y), r = s - q d
// exact by FMA, RN(q + r y) = RN(s / d) when nothing under/overflows): three
// dependent FP64 ops instead of the division subroutine on the critical path.
// Outside the safe exponent range (and for s == 0, to keep the sign of a
// zero) the IEEE division runs.
__device__ __forceinline__ double gp_div(double s, double d, double y, bool fast_ok) {
  const double as = fabs(s);
  if (fast_ok && as < 0x1p900 && (as > 0x1p-900 || as == 0.0)) {
    const double q = s * y;
    const double r = __fma_rn(-q, d, s);
    const double q2 = __fma_rn(r, y, q);
    return as == 0.0 ? s : q2;  // 0 / d = 0 with the sign of s (d > 0)
  }
  return s / d;
}

// n_train <= 1024: one WARP per query point (W warps per CTA), no block
// barrier in the loop.  Lane l owns rows l, l+32, ... (RM = ceil(n/32)
// registers); step j: every lane divides the owner's s_j (v_j = s_j / L[j][j],
// gp.cpp:201), every row i > j subtracts L[i][j] v_j (gp.cpp:200) — the
// reference's j order per row.  mean and the variance accumulate in the same
// j order (gp.cpp:193-194, 204-205).  L streams through a shared-memory ring
// in CHUNKS of C columns (one 1D bulk copy and one mbarrier wait per chunk);
// thread 0 refills the chunk released one chunk earlier.  The C steps of a
// chunk are unrolled and branch-free: the columns are padded to a multiple of
// C with identity steps (L column 0, diagonal 1, k* = alpha = 0, so s, mean
// and the variance keep their bits), so a chunk never tests j < n.
template <int RM>
struct GpRing {
  static constexpr int cols = RM >= 32 ? 4 : 8;  // <= 32 KB chunks
  static constexpr int depth = 4;
  static constexpr int lag = 2;
};

template <int RM>
__global__ void __launch_bounds__(128) k_gp_ring(
    const double* __restrict__ kstar, int n, int ldt, int64_t P,
    const double* __restrict__ alpha, const double* __restrict__ lt,
    const double* __restrict__ diag, const double* __restrict__ rdiag, int fast_ok,
    double signal_var, double noise_var, double confidence, double* __restrict__ out_a,
    double* __restrict__ out_b, int bounds) {
  extern __shared__ __align__(16) unsigned char gsm[];
  constexpr int C = GpRing<RM>::cols, D = GpRing<RM>::depth, LAG = GpRing<RM>::lag;
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npad = (n + C - 1) / C * C;  // <= ldt
  double* ring = reinterpret_cast<double*>(gsm);  // D chunks of C columns
  double* sal = ring + D * C * ldt;
  double* sdg = sal + ldt;
  double* srd = sdg + ldt;
  double* sks = srd + ldt + w * ldt;
  uint64_t* full = reinterpret_cast<uint64_t*>(srd + ldt + W * ldt);
  uint64_t* empty = full + D;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * W + w;
  const bool live = p < P;
  const int nchunks = npad / C;
  if (threadIdx.x == 0) {
    for (int k = 0; k < D; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gp_smem(full + k)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(gp_smem(empty + k)), "r"(W));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < ldt; i += blockDim.x) {
    sal[i] = i < n ? alpha[i] : 0.0;
    sdg[i] = i < n ? diag[i] : 1.0;
    srd[i] = i < n ? rdiag[i] : 1.0;
  }
  for (int i = lane; i < ldt; i += 32) sks[i] = (live && i < n) ? kstar[p * n + i] : 0.0;
  __syncthreads();
  const uint32_t chunkb = static_cast<uint32_t>(C) * static_cast<uint32_t>(ldt) * 8u;
  if (threadIdx.x == 0)
    for (int c = 0; c < D && c < nchunks; ++c)
      gp_column(gp_smem(ring + c * C * ldt), lt + static_cast<size_t>(c) * C * ldt, chunkb,
                gp_smem(full + c));
  const bool fok = fast_ok != 0;
  // rows >= n hold 0 and their L entries are 0 (ldt = 32 RM): no row masks
  double s[RM];
#pragma unroll
  for (int k = 0; k < RM; ++k) s[k] = sks[lane + 32 * k];
  double mean = 0.0, var = signal_var;
#pragma unroll
  for (int kb = 0; kb < RM; ++kb) {
    for (int cb = 0; cb < 32 / C; ++cb) {
      const int j0 = kb * 32 + cb * C;
      if (j0 >= npad) break;  // CTA-uniform, once per chunk
      const int c = j0 / C;
      gp_wait(gp_smem(full + c % D), static_cast<uint32_t>(c / D) & 1u);
      const double* col = ring + (c % D) * C * ldt + lane;
#pragma unroll
      for (int u = 0; u < C; ++u) {
        const int lj = cb * C + u, j = j0 + u;
        // every lane divides the owner's s_j (warp-uniform values and branch)
        const double sj = __shfl_sync(0xffffffffu, s[kb], lj);
        const double vj = gp_div(sj, sdg[j], srd[j], fok);
        const double* cc = col + u * ldt;
        {
          const double upd = s[kb] - cc[32 * kb] * vj;
          s[kb] = lane > lj ? upd : (lane == lj ? vj : s[kb]);
        }
#pragma unroll
        for (int k = kb + 1; k < RM; ++k) s[k] = s[k] - cc[32 * k] * vj;
        mean += sks[j] * sal[j];
        var -= vj * vj;
      }
      // chunk done: release it, refill the one released a chunk earlier
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(gp_smem(empty + c % D))
                     : "memory");
      const int cr = c - LAG + 1;
      if (threadIdx.x == 0 && cr >= 0 && cr + D < nchunks) {
        gp_wait(gp_smem(empty + cr % D), static_cast<uint32_t>(cr / D) & 1u);
        gp_column(gp_smem(ring + (cr % D) * C * ldt), lt + static_cast<size_t>(cr + D) * C * ldt,
                  chunkb, gp_smem(full + cr % D));
      }
    }
  }
  if (live && lane == 0) {
    var = var < 0.0 ? 0.0 : var;  // std::max(var, 0.0)
    if (bounds) {                 // gp.cpp:241-245
      const double band = confidence * sqrt(var + noise_var);
      out_a[p] = mean - band;
      out_b[p] = mean + band;
    } else {
      out_a[p] = mean;
      out_b[p] = var;
    }
  }
}

// row-major chol -> column-major strictly-lower part (leading dim ldt,
// zero-padded) + diagonal
__global__ void k_gp_prep(const double* __restrict__ chol, int n, int ncols, int ldt,
                          double* __restrict__ lt, double* __restrict__ diag,
                          double* __restrict__ rdiag) {
  const int64_t total = static_cast<int64_t>(ncols) * ldt;  // columns >= n: zero
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / ldt, i = e - j * ldt;  // lt[j*ldt + i] = L[i][j]
    lt[e] = (i > j && i < n && j < n) ? chol[i * n + j] : 0.0;
    if (i == j && i < n) {
      diag[i] = chol[i * n + i];
      rdiag[i] = 1.0 / chol[i * n + i];  // IEEE (-prec-div=true): RN(1/d)
    }
  }
}

// lo/hi of every node from its input point's entry: m(node) = sum over grid
// axes of idx_a * wgt_a (wgt: the point-enumeration strides of the axes in
// input_dims, summed when an axis appears twice).
__global__ void k_gp_broadcast(DevGrid g, uint32_t wgt0, uint32_t wgt1, uint32_t wgt2,
                               uint32_t wgt3, uint32_t wgt4, uint32_t wgt5,
                               const double* __restrict__ tlo, const double* __restrict__ thi,
                               double* __restrict__ lo, double* __restrict__ hi) {
  const uint32_t wg[kMaxDims] = {wgt0, wgt1, wgt2, wgt3, wgt4, wgt5};
  for (uint32_t lin = blockIdx.x * blockDim.x + threadIdx.x; lin < g.size;
       lin += gridDim.x * blockDim.x) {
    uint32_t rest = lin, m = 0;
    for (int d = g.nd - 1; d >= 0; --d) {
      const uint32_t q = g.divs[d].quo(rest);
      m += (rest - q * g.n[d]) * wg[d];
      rest = q;
    }
    lo[lin] = __ldg(tlo + m);
    hi[lin] = __ldg(thi + m);
  }
}

// Same, one warp per row of the contiguous last axis (rows = size / n_last):
// the row's table offset is unravelled once, lanes store consecutive nodes
// (coalesced), so the kernel runs at the HBM write rate.
__global__ void k_gp_broadcast_rows(DevGrid g, uint32_t wgt0, uint32_t wgt1, uint32_t wgt2,
                                    uint32_t wgt3, uint32_t wgt4, uint32_t wgt5,
                                    const double* __restrict__ tlo,
                                    const double* __restrict__ thi, double* __restrict__ lo,
                                    double* __restrict__ hi) {
  const uint32_t wg[kMaxDims] = {wgt0, wgt1, wgt2, wgt3, wgt4, wgt5};
  const int last = g.nd - 1;
  const uint32_t nl = g.n[last], wl = wg[last];
  const uint32_t rows = g.size / nl;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += nw) {
    uint32_t rest = row, m = 0;
    for (int d = last - 1; d >= 0; --d) {
      const uint32_t q = g.divs[d].quo(rest);
      m += (rest - q * g.n[d]) * wg[d];
      rest = q;
    }
    const size_t base = static_cast<size_t>(row) * nl;
    for (uint32_t i = lane; i < nl; i += 32) {
      const uint32_t mi = m + i * wl;
      lo[base + i] = __ldg(tlo + mi);
      hi[base + i] = __ldg(thi + mi);
    }
  }
}

double coord_of(const DevGrid& g, int d, uint32_t k) {  // grid.cpp:33-38
  if (k == g.n[d] - 1) return g.max[d];
  return g.min[d] + static_cast<double>(k) * g.spacing[d];
}

int check_model(const hjb_gp_model& m, const char* who) {
  if (m.input_dim < 1 || m.input_dim > HJB_MAX_DIMS)
    return set_err(HJB_ERR_INVALID_ARGUMENT, std::string(who) + ": GP input dim out of range");
  if (m.n_train < 0 || m.n_train > 8192)
    return set_err(HJB_ERR_UNSUPPORTED, std::string(who) + ": GP training count must be 0..8192");
  if (m.n_train > 0 && (!m.inputs || !m.alpha || !m.chol))
    return set_err(HJB_ERR_INVALID_ARGUMENT, std::string(who) + ": GP factor pointers null");
  for (int d = 0; d < m.input_dim; ++d)
    if (!(m.lengthscales[d] > 0.0))
      return set_err(HJB_ERR_INVALID_ARGUMENT, "GP: lengthscales must be > 0");
  if (!(m.signal_var > 0.0))
    return set_err(HJB_ERR_INVALID_ARGUMENT, "GP: signal variance must be > 0");
  if (!(m.noise_var >= 0.0))
    return set_err(HJB_ERR_INVALID_ARGUMENT, "GP: noise variance must be >= 0");
  return HJB_OK;
}

// k*(x_p, x_i) for P points (x: P x input_dim) — GpModel::kernel, gp.cpp:22-30
void tabulate_kstar(const hjb_gp_model& m, int64_t P, const double* x, double* out) {
  const int64_t n = m.n_train;
  const int dim = m.input_dim;
  auto work = [&](int64_t p0, int64_t p1) {
    for (int64_t p = p0; p < p1; ++p) {
      const double* a = x + p * dim;
      for (int64_t i = 0; i < n; ++i) {
        const double* b = m.inputs + i * dim;
        double q = 0.0;
        for (int d = 0; d < dim; ++d) {
          const double r = (a[d] - b[d]) / m.lengthscales[d];
          q += r * r;
        }
        out[p * n + i] = m.signal_var * std::exp(-0.5 * q);
      }
    }
  };
  const int64_t evals = P * n;
  unsigned th = std::thread::hardware_concurrency();
  if (th == 0) th = 1;
  if (evals < (1 << 16) || th == 1) {
    work(0, P);
    return;
  }
  th = static_cast<unsigned>(std::min<int64_t>(th, P));
  std::vector<std::thread> pool;
  const int64_t per = (P + th - 1) / th;
  for (unsigned k = 0; k < th; ++k) {
    const int64_t a = k * per, b = std::min<int64_t>(P, a + per);
    if (a < b) pool.emplace_back(work, a, b);
  }
  for (auto& t : pool) t.join();
}

// posterior over P points on the device: bounds ? (lo, hi) : (mean, var)
int posterior(hjb_context* ctx, const hjb_gp_model& m, int64_t P, const double* x,
              double confidence, int bounds, double* out_a_dev, double* out_b_dev) {
  const int64_t n = m.n_train;
  if (n == 0) {  // GpModel::prior: {0, signal_var} (gp.cpp:190)
    double a, b;
    if (bounds) {
      const double band = confidence * std::sqrt(m.signal_var + m.noise_var);
      a = 0.0 - band;
      b = 0.0 + band;
    } else {
      a = 0.0;
      b = m.signal_var;
    }
    std::vector<double> ha(P, a), hb(P, b);
    CUDA_TRY(cudaMemcpyAsync(out_a_dev, ha.data(), P * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(out_b_dev, hb.data(), P * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return HJB_OK;
  }
  // device buffers of the context (grow-only): k*, raw factor, its
  // column-major copy, diagonal, alpha
  std::vector<double> ks(static_cast<size_t>(P) * n);
  tabulate_kstar(m, P, x, ks.data());
  const size_t nn = static_cast<size_t>(n) * n;
  // column stride: 32 * ceil(n/32) for the warp kernel (no row masks), else
  // n rounded to 16 bytes
  const int rm = n <= 32 ? 1 : n <= 64 ? 2 : n <= 128 ? 4 : n <= 256 ? 8 : n <= 512 ? 16 : 32;
  const int ldt = static_cast<int>(n <= 1024 ? 32 * rm : (n + 1) / 2 * 2);
  const int ncols = static_cast<int>((n + 7) / 8 * 8);  // chunk padding (zero columns)
  const size_t ntl = static_cast<size_t>(ncols) * ldt;
  auto al = [](size_t x) { return (x + 31) / 32 * 32; };  // 256-byte sub-buffers
  CUDA_TRY(ctx->gpa.ensure(ks.size() * sizeof(double)));
  CUDA_TRY(ctx->gpb.ensure((al(nn) + al(ntl) + 3 * al(n)) * sizeof(double)));
  double* dks = ctx->gpa.d();
  double* draw = ctx->gpb.d();
  double* dlt = draw + al(nn);
  double* ddg = dlt + al(ntl);
  double* drd = ddg + al(n);
  double* dal = drd + al(n);
  CUDA_TRY(cudaMemcpyAsync(dks, ks.data(), ks.size() * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(draw, m.chol, nn * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(dal, m.alpha, n * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  const int sms = sm_count(ctx->device);
  k_gp_prep<<<static_cast<unsigned>(std::min<size_t>((ntl + 255) / 256, 4u * sms)), 256, 0,
              ctx->stream>>>(draw, static_cast<int>(n), ncols, ldt, dlt, ddg, drd);
  CUDA_TRY(cudaGetLastError());
  ++ctx->launches;
  // Markstein division is exact while the diagonal stays in a safe range
  bool fast_ok = true;
  for (int64_t i = 0; i < n; ++i) {
    const double d = std::fabs(m.chol[i * n + i]);
    if (!(d > 0x1p-100 && d < 0x1p100)) fast_ok = false;
  }
  if (n <= 1024) {
    const int W = 4;
    const unsigned blocks = static_cast<unsigned>((P + W - 1) / W);
    const int ringcols = rm >= 32 ? GpRing<32>::depth * GpRing<32>::cols
                         : rm >= 16 ? GpRing<16>::depth * GpRing<16>::cols
                                    : GpRing<1>::depth * GpRing<1>::cols;
    const size_t smem = static_cast<size_t>(ringcols + 3 + W) * ldt * sizeof(double) +
                        2 * GpRing<1>::depth * sizeof(uint64_t);
#define HJB_GPW(R)                                                                          \
  do {                                                                                      \
    CUDA_TRY(cudaFuncSetAttribute(k_gp_ring<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  static_cast<int>(smem)));                                 \
    k_gp_ring<R><<<blocks, 32 * W, smem, ctx->stream>>>(                                    \
        dks, static_cast<int>(n), ldt, P, dal, dlt, ddg, drd, fast_ok ? 1 : 0, m.signal_var, \
        m.noise_var,                                                                        \
        confidence, out_a_dev, out_b_dev, bounds);                                          \
  } while (0)
    switch (rm) {
      case 1: HJB_GPW(1); break;
      case 2: HJB_GPW(2); break;
      case 4: HJB_GPW(4); break;
      case 8: HJB_GPW(8); break;
      case 16: HJB_GPW(16); break;
      default: HJB_GPW(32); break;
    }
#undef HJB_GPW
    CUDA_TRY(cudaGetLastError());
    ++ctx->launches;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // host staging buffers die here
    return HJB_OK;
  }
  const int R = n <= 2048 ? 2 : n <= 4096 ? 4 : 8;
  const int T = static_cast<int>(std::min<int64_t>(1024, ((n + R - 1) / R + 31) / 32 * 32));
  const size_t smem = n * sizeof(double);
  for (int64_t p0 = 0; p0 < P; p0 += 65535) {
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(65535, P - p0));
    const double* kp = dks + p0 * n;
    double* oa = out_a_dev + p0;
    double* ob = out_b_dev + p0;
#define HJB_GP_LAUNCH(RR)                                                                    \
  do {                                                                                       \
    if (smem > 48 * 1024)                                                                    \
      CUDA_TRY(cudaFuncSetAttribute(k_gp_posterior<RR>,                                      \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_gp_posterior<RR><<<blocks, T, smem, ctx->stream>>>(kp, (int)n, dal, dlt, ldt, ddg,          \
                                                         m.signal_var, m.noise_var,          \
                                                         confidence, oa, ob, bounds);        \
  } while (0)
    switch (R) {
      case 2: HJB_GP_LAUNCH(2); break;
      case 4: HJB_GP_LAUNCH(4); break;
      default: HJB_GP_LAUNCH(8); break;
    }
#undef HJB_GP_LAUNCH
    CUDA_TRY(cudaGetLastError());
    ++ctx->launches;
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // host staging buffers die here
  return HJB_OK;
}

// ---------------------------------------------------------------- fit
// GpModel::fit (gp.cpp:124-186) on the host: O(n^3) once per update, off the
// per-node path.  Same subsample, candidate grid, jitter and LML as the
// reference; the Cholesky is the textbook left-looking LLT (Eigen, which the
// reference uses, is not available here), so factors agree with Eigen's to
// rounding, not bitwise — bounds_on_grid is bitwise GIVEN the factor.

// evenly spaced subsample keeping first and last (gp.cpp:43-56)
std::vector<int64_t> uniform_subsample(int64_t n, int64_t cap) {
  std::vector<int64_t> idx;
  if (n <= cap) {
    idx.resize(n);
    for (int64_t i = 0; i < n; ++i) idx[i] = i;
    return idx;
  }
  idx.reserve(cap);
  for (int64_t i = 0; i < cap; ++i) idx.push_back((i * (n - 1)) / (cap - 1));
  idx.erase(std::unique(idx.begin(), idx.end()), idx.end());
  return idx;
}

struct Hp {
  double sf, sn;
  std::vector<double> ls;
};

struct Factor {
  std::vector<double> L, alpha;
  double lml = 0.0;
  bool ok = false;
};

// factorize (gp.cpp:64-96): K + (noise + 1e-8 sf) I = L L^T, alpha, LML
Factor factorize(const std::vector<const double*>& xs, int dim, const std::vector<double>& y,
                 const Hp& hp) {
  const int64_t n = static_cast<int64_t>(xs.size());
  std::vector<double> k(n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      double q = 0.0;
      for (int d = 0; d < dim; ++d) {
        const double r = (xs[i][d] - xs[j][d]) / hp.ls[d];
        q += r * r;
      }
      const double v = hp.sf * std::exp(-0.5 * q);
      k[i * n + j] = v;
      k[j * n + i] = v;
    }
  const double jitter = 1e-8 * hp.sf;
  for (int64_t i = 0; i < n; ++i) k[i * n + i] += hp.sn + jitter;
  Factor f;
  f.L.assign(n * n, 0.0);
  for (int64_t j = 0; j < n; ++j) {
    double d = k[j * n + j];
    for (int64_t p = 0; p < j; ++p) d -= f.L[j * n + p] * f.L[j * n + p];
    if (!(d > 0.0)) return f;  // not positive definite
    const double ljj = std::sqrt(d);
    f.L[j * n + j] = ljj;
    for (int64_t i = j + 1; i < n; ++i) {
      double s = k[i * n + j];
      for (int64_t p = 0; p < j; ++p) s -= f.L[i * n + p] * f.L[j * n + p];
      f.L[i * n + j] = s / ljj;
    }
  }
  // alpha = L^-T L^-1 y
  std::vector<double> z(n);
  for (int64_t i = 0; i < n; ++i) {
    double s = y[i];
    for (int64_t p = 0; p < i; ++p) s -= f.L[i * n + p] * z[p];
    z[i] = s / f.L[i * n + i];
  }
  f.alpha.assign(n, 0.0);
  for (int64_t i = n; i-- > 0;) {
    double s = z[i];
    for (int64_t p = i + 1; p < n; ++p) s -= f.L[p * n + i] * f.alpha[p];
    f.alpha[i] = s / f.L[i * n + i];
  }
  double quad = 0.0;
  for (int64_t i = 0; i < n; ++i) quad += y[i] * f.alpha[i];
  double logdet = 0.0;
  for (int64_t i = 0; i < n; ++i) logdet += std::log(f.L[i * n + i]);
  f.lml = -0.5 * quad - logdet - 0.5 * static_cast<double>(n) * std::log(2.0 * M_PI);
  f.ok = true;
  return f;
}

// candidate_grid (gp.cpp:98-122)
std::vector<Hp> candidate_grid(const std::vector<const double*>& xs, int dim,
                               const std::vector<double>& y) {
  double sq = 0.0;
  for (double v : y) sq += v * v;
  const double y_sd =
      std::max(std::sqrt(sq / static_cast<double>(y.size()) + 1e-12), 1e-3);
  std::vector<double> range(dim, 1.0);
  for (int d = 0; d < dim; ++d) {
    double lo = xs[0][d], hi = xs[0][d];
    for (const double* x : xs) {
      lo = std::min(lo, x[d]);
      hi = std::max(hi, x[d]);
    }
    range[d] = std::max(hi - lo, 1e-3);
  }
  std::vector<Hp> out;
  for (double sf : {0.5, 1.0, 2.0})
    for (double ls : {0.08, 0.2, 0.5, 1.0})
      for (double sn : {0.03, 0.08, 0.2, 0.5}) {
        Hp hp;
        hp.sf = (sf * y_sd) * (sf * y_sd);
        hp.ls.assign(dim, 0.0);
        for (int d = 0; d < dim; ++d) hp.ls[d] = ls * range[d];
        hp.sn = (sn * y_sd) * (sn * y_sd);
        out.push_back(hp);
      }
  return out;
}

}  // namespace
}  // namespace hjb

using namespace hjb;

int hjb_gp_fit(int64_t n, int32_t input_dim, const double* x, const double* y,
               const hjb_gp_fit_config* cfg, double* inputs_out, double* alpha_out,
               double* chol_out, hjb_gp_model* model_out, double* lml_out) {
  if (n <= 0) return set_err(HJB_ERR_INVALID_ARGUMENT, "GP fit: need at least one measurement");
  if (!x || !y || !cfg || !model_out)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "GP fit: null argument");
  if (input_dim < 1 || input_dim > HJB_MAX_DIMS)
    return set_err(HJB_ERR_UNSUPPORTED, "GP fit: input dim out of range");
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < input_dim; ++d)
      if (!std::isfinite(x[i * input_dim + d]))
        return set_err(HJB_ERR_INVALID_ARGUMENT, "GP fit: non-finite input");
    if (!std::isfinite(y[i])) return set_err(HJB_ERR_INVALID_ARGUMENT, "GP fit: non-finite value");
  }
  if (cfg->max_training < 2 || cfg->search_subsample < 2)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "GP fit: subsample caps must be >= 2");
  const auto train = uniform_subsample(n, cfg->max_training);
  std::vector<const double*> xs;
  std::vector<double> ys;
  for (int64_t i : train) {
    xs.push_back(x + i * input_dim);
    ys.push_back(y[i]);
  }
  Hp chosen{cfg->prior_signal_var, cfg->prior_noise_var, {}};
  for (int d = 0; d < cfg->prior_n_lengthscales; ++d)  // a count > HJB_MAX_DIMS never matches
    chosen.ls.push_back(d < HJB_MAX_DIMS ? cfg->prior_lengthscales[d] : 1.0);
  auto validate = [&](const Hp& hp) -> int {  // GpHyperparams::validate, gp.cpp:14-21
    if (!(hp.sf > 0.0)) return set_err(HJB_ERR_INVALID_ARGUMENT, "GP: signal variance must be > 0");
    if (!(hp.sn >= 0.0)) return set_err(HJB_ERR_INVALID_ARGUMENT, "GP: noise variance must be >= 0");
    if (static_cast<int>(hp.ls.size()) != input_dim)
      return set_err(HJB_ERR_INVALID_ARGUMENT, "GP: lengthscale count does not match input dim");
    for (double l : hp.ls)
      if (!(l > 0.0)) return set_err(HJB_ERR_INVALID_ARGUMENT, "GP: lengthscales must be > 0");
    return HJB_OK;
  };
  int rc;
  if (cfg->policy == HJB_GP_SEARCH) {
    const auto sidx = uniform_subsample(static_cast<int64_t>(xs.size()), cfg->search_subsample);
    std::vector<const double*> sx;
    std::vector<double> sy;
    for (int64_t i : sidx) {
      sx.push_back(xs[i]);
      sy.push_back(ys[i]);
    }
    double best = -INFINITY;
    for (const Hp& hp : candidate_grid(sx, input_dim, sy)) {
      const Factor fr = factorize(sx, input_dim, sy, hp);
      if (fr.ok && fr.lml > best) {
        best = fr.lml;
        chosen = hp;
      }
    }
  } else if ((rc = validate(chosen))) {
    return rc;
  }
  if (static_cast<int>(chosen.ls.size()) != input_dim)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "GP fit: fixed hyperparams do not match input dim");
  const Factor fr = factorize(xs, input_dim, ys, chosen);
  if (!fr.ok) return set_err(HJB_ERR_RUNTIME, "GP fit: kernel matrix singular after jitter");
  const int64_t m = static_cast<int64_t>(xs.size());
  if (inputs_out)
    for (int64_t i = 0; i < m; ++i)
      std::memcpy(inputs_out + i * input_dim, xs[i], input_dim * sizeof(double));
  if (alpha_out) std::memcpy(alpha_out, fr.alpha.data(), m * sizeof(double));
  if (chol_out) std::memcpy(chol_out, fr.L.data(), m * m * sizeof(double));
  std::memset(model_out, 0, sizeof *model_out);
  model_out->input_dim = input_dim;
  model_out->n_dims = input_dim;
  for (int d = 0; d < input_dim; ++d) model_out->input_dims[d] = d;
  model_out->n_train = m;
  model_out->signal_var = chosen.sf;
  model_out->noise_var = chosen.sn;
  for (int d = 0; d < input_dim; ++d) model_out->lengthscales[d] = chosen.ls[d];
  model_out->inputs = inputs_out;
  model_out->alpha = alpha_out;
  model_out->chol = chol_out;
  if (lml_out) *lml_out = fr.lml;
  return HJB_OK;
}

int hjb_gp_bounds_on_grid_dev(hjb_context* ctx, const hjb_grid* gi, int32_t channels,
                              const hjb_gp_model* models, double confidence,
                              double* const* lo_out, double* const* hi_out) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  DevGrid g;
  if ((rc = make_grid(gi, g))) return rc;
  if (channels < 0 || channels > HJB_MAX_INPUT || (channels > 0 && (!models || !lo_out || !hi_out)))
    return set_err(HJB_ERR_INVALID_ARGUMENT, "bounds_on_grid: one input-dim map per channel");
  for (int ch = 0; ch < channels; ++ch) {
    const hjb_gp_model& m = models[ch];
    if (m.n_dims != m.input_dim)
      return set_err(HJB_ERR_INVALID_ARGUMENT,
                     "bounds_on_grid: input-dim map does not match GP");
    if ((rc = check_model(m, "bounds_on_grid"))) return rc;
    for (int d = 0; d < m.n_dims; ++d)
      if (m.input_dims[d] < 0 || m.input_dims[d] >= g.nd)
        return set_err(HJB_ERR_INVALID_ARGUMENT,
                       "bounds_on_grid: input dim out of grid range");
    if (!lo_out[ch] || !hi_out[ch])
      return set_err(HJB_ERR_INVALID_ARGUMENT, "bounds_on_grid: null output");
  }
  for (int ch = 0; ch < channels; ++ch) {
    const hjb_gp_model& m = models[ch];
    // distinct inputs: odometer over the input dims, last fastest
    const int D = m.n_dims;
    int64_t M = 1;
    uint32_t mstride[kMaxDims];
    for (int d = D - 1; d >= 0; --d) {
      mstride[d] = static_cast<uint32_t>(M);
      M *= g.n[m.input_dims[d]];
    }
    if (M > (int64_t(1) << 26))
      return set_err(HJB_ERR_UNSUPPORTED, "bounds_on_grid: too many distinct GP inputs");
    std::vector<double> xs(static_cast<size_t>(M) * D);
    for (int64_t p = 0; p < M; ++p)
      for (int d = 0; d < D; ++d) {
        const uint32_t k = static_cast<uint32_t>((p / mstride[d]) % g.n[m.input_dims[d]]);
        xs[p * D + d] = coord_of(g, m.input_dims[d], k);
      }
    CUDA_TRY(ctx->gpc.ensure(2 * M * sizeof(double)));
    double* tab = ctx->gpc.d();
    if ((rc = posterior(ctx, m, M, xs.data(), confidence, 1, tab, tab + M))) return rc;
    uint32_t wg[kMaxDims] = {0, 0, 0, 0, 0, 0};
    for (int d = 0; d < D; ++d) wg[m.input_dims[d]] += mstride[d];
    const int sms = sm_count(ctx->device);
    const unsigned blocks =
        static_cast<unsigned>(std::min<uint64_t>((g.size + 255) / 256, 8ull * sms));
    if (g.nd >= 2 && g.n[g.nd - 1] <= 256)
      k_gp_broadcast_rows<<<8u * sms, 256, 0, ctx->stream>>>(g, wg[0], wg[1], wg[2], wg[3], wg[4],
                                                             wg[5], tab, tab + M, lo_out[ch],
                                                             hi_out[ch]);
    else
      k_gp_broadcast<<<blocks, 256, 0, ctx->stream>>>(g, wg[0], wg[1], wg[2], wg[3], wg[4], wg[5],
                                                      tab, tab + M, lo_out[ch], hi_out[ch]);
    CUDA_TRY(cudaGetLastError());
    ++ctx->launches;
  }
  return HJB_OK;
}

int hjb_gp_bounds_on_grid(hjb_context* ctx, const hjb_grid* gi, int32_t channels,
                          const hjb_gp_model* models, double confidence, double* const* lo_out,
                          double* const* hi_out) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  DevGrid g;
  if ((rc = make_grid(gi, g))) return rc;
  if (channels < 0 || channels > HJB_MAX_INPUT || (channels > 0 && (!lo_out || !hi_out)))
    return set_err(HJB_ERR_INVALID_ARGUMENT, "bounds_on_grid: one input-dim map per channel");
  const size_t bytes = static_cast<size_t>(g.size) * sizeof(double);
  DevBuf buf;
  CUDA_TRY(buf.ensure(2 * channels * bytes + 8));
  double* lo[HJB_MAX_INPUT] = {nullptr, nullptr, nullptr};
  double* hi[HJB_MAX_INPUT] = {nullptr, nullptr, nullptr};
  for (int ch = 0; ch < channels; ++ch) {
    lo[ch] = buf.d() + 2 * ch * static_cast<size_t>(g.size);
    hi[ch] = lo[ch] + g.size;
  }
  if ((rc = hjb_gp_bounds_on_grid_dev(ctx, gi, channels, models, confidence, lo, hi))) return rc;
  for (int ch = 0; ch < channels; ++ch) {
    CUDA_TRY(cudaMemcpyAsync(lo_out[ch], lo[ch], bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(hi_out[ch], hi[ch], bytes, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return HJB_OK;
}

int hjb_gp_predict_batch(hjb_context* ctx, const hjb_gp_model* model, int64_t nq,
                         const double* x, double* mean, double* variance) {
  int rc;
  if ((rc = check_ctx(ctx))) return rc;
  if (!model) return set_err(HJB_ERR_INVALID_ARGUMENT, "GP predict: null model");
  if ((rc = check_model(*model, "GP predict"))) return rc;
  if (nq < 0 || (nq > 0 && (!x || !mean || !variance)))
    return set_err(HJB_ERR_INVALID_ARGUMENT, "GP predict: bad batch");
  if (nq == 0) return HJB_OK;
  CUDA_TRY(ctx->gpc.ensure(2 * nq * sizeof(double)));
  double* out = ctx->gpc.d();
  if ((rc = posterior(ctx, *model, nq, x, 0.0, 0, out, out + nq))) return rc;
  CUDA_TRY(cudaMemcpyAsync(mean, out, nq * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(variance, out + nq, nq * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return HJB_OK;
}
