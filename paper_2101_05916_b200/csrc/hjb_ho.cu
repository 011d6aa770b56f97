// hjb_ho.cu — high-order (ENO2/ENO3 + TVD-RK2/RK3) solve and single step.
//
// No reference implementation exists (reference SPEC.md:324 lists
// high-order schemes as non-goals); the scheme is the repo's own CPU
// restatement (oracle/hj_oracle.c, "high order" section), reproduced bit
// for bit by k_ho_stage.  One stage = one HBM pass: it reads the stage input
// (stencil), V_n and c, and writes the clamped stage output.  The loop runs
// on the device like the first-order solve: a WHILE-conditional graph whose
// body holds the stages of several steps; the last stage of a step runs the
// solve() epilogue (residual = max|V_{n+1} - V_n| / dt).
#include <cstring>
#include <string>

#include <cstdlib>

#include "hjb_fast4d.cuh"
#include "hjb_ho.cuh"
#include "hjb_internal.cuh"
#include "hjb_kernels.cuh"

namespace hjb {

namespace {

int scheme_id(const hjb_solve_config* cfg) {
  if (cfg->scheme == HJB_GODUNOV) return kGodunov;
  return cfg->dissipation == HJB_GLOBAL ? kLfGlobal : kLfPerNode;
}

StepArgs ho_args(const DevGrid& g, const DevModel& m, const double* c, double dt,
                 const double* galpha, const hjb_solve_config* cfg) {
  StepArgs a;
  std::memset(&a, 0, sizeof a);
  a.g = g;
  a.m = m;
  a.c = c;
  a.dt = dt;
  a.scheme = scheme_id(cfg);
  for (int d = 0; d < kMaxDims; ++d) a.galpha[d] = galpha[d];
  a.order = cfg->spatial_order < 1 ? 1 : cfg->spatial_order;
  a.target = cfg->target;  // reach-avoid: every stage min(l, .) then the clamp
  return a;
}

// stage table of a TVD-RK step: (src_sel, dst_sel, kind)
struct Stage {
  int src, dst, kind;
};

int stages_of(int rk, Stage* st) {
  if (rk <= 1) {
    st[0] = {0, 0, 0};
    return 1;
  }
  if (rk == 2) {
    st[0] = {0, 1, 0};
    st[1] = {1, 0, 1};
    return 2;
  }
  st[0] = {0, 1, 0};
  st[1] = {1, 2, 2};
  st[2] = {2, 0, 3};
  return 3;
}

}  // namespace

int ho_solve(hjb_context* ctx, const DevGrid& g, const DevModel& m, const double* init,
             const double* c, const hjb_solve_config* cfg, double dt, const double* galpha,
             double* out, hjb_solve_result* res) {
  if (g.nd > 4) return set_err(HJB_ERR_UNSUPPORTED, "solve: high-order schemes up to rank 4");
  const size_t bytes = static_cast<size_t>(g.size) * sizeof(double);
  // 4D fast-path models (Godunov, constant bounds): padded layout + k_ho4d
  const char* fe = std::getenv("HJB_FAST");
  int shape = (fe && std::strcmp(fe, "0") == 0) ? -1 : fast4d_shape(g, m, scheme_id(cfg));
  if (cfg->target) shape = -1;  // target sets run the generic stage kernel
  // run-time row shapes: k_ho4t<ShapeGen> unless a row depends on x0 (the
  // march axis of the stage kernels keeps its slopes loop invariant)
  Fast4dArgs gr;
  std::memset(&gr, 0, sizeof gr);
  if (shape == kShapeGen) {
    fast4d_gen_rows(m, gr);
    if (gr.gx0) shape = -1;
  }
  if (shape >= 0 && scheme_id(cfg) != kGodunov) {
    // Lax-Friedrichs runs only in the TMA-staged kernel (k_ho4t)
    Ho4dArgs t;
    std::memset(&t, 0, sizeof t);
    t.order = cfg->spatial_order > 3 ? 3 : (cfg->spatial_order < 1 ? 1 : cfg->spatial_order);
    t.lf = 1;
    t.gen = shape == kShapeGen ? 1 : 0;
    ho4d_config(g, sm_count(ctx->device), t);
    if (!t.tma) shape = -1;
  }
  // the 4D kernel's configuration fixes the stage-buffer layout (padded, or
  // with ghost cells for k_eno3g)
  Ho4dArgs h4;
  std::memset(&h4, 0, sizeof h4);
  if (shape >= 0) {
    h4.order = cfg->spatial_order > 3 ? 3 : (cfg->spatial_order < 1 ? 1 : cfg->spatial_order);
    fill_lf(m, scheme_id(cfg), galpha, h4.lf, h4.lp);
    if (shape == kShapeGen) {
      h4.gen = 1;
      for (int d = 0; d < 4; ++d) {
        h4.gax[d] = gr.gax[d];
        h4.gbx[d] = gr.gbx[d];
      }
      h4.glin = gr.glin;
    }
    ho4d_config(g, sm_count(ctx->device), h4);
    if (shape == kShapeGen && !h4.tma) {  // no TMA configuration: the generic stage kernel
      shape = -1;
      std::memset(&h4, 0, sizeof h4);
    }
  }
  const size_t pbytes = shape >= 0 ? g.n[0] * ho4d_plane(h4) * sizeof(double) : bytes;
  CUDA_TRY(ctx->v0.ensure(pbytes));
  CUDA_TRY(ctx->v1.ensure(pbytes));
  CUDA_TRY(ctx->v2.ensure(pbytes));
  CUDA_TRY(ctx->v3.ensure(pbytes));
  if (shape >= 0) {
    CUDA_TRY(ctx->pcbuf.ensure(pbytes));
    CUDA_TRY(ho4d_pad(init, ctx->v0.d(), g.n[0], h4, ctx->stream));
    ++ctx->launches;
    int rcp;
    if (h4.eno3g && !h4.lf &&
        (rcp = constraint_planes(ctx, g, c, &h4.cplane, g.size >= kSustainedCells)))
      return rcp;
    if (!h4.cplane) {
      CUDA_TRY(ho4d_pad(c, ctx->pcbuf.d(), g.n[0], h4, ctx->stream));
      ++ctx->launches;
    }
  } else {
    CUDA_TRY(cudaMemcpyAsync(ctx->v0.p, init, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (cfg->max_iters == 0) {
    if (out != init)
      CUDA_TRY(cudaMemcpyAsync(out, init, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return HJB_OK;
  }
  const long long cap =
      std::min<long long>(cfg->max_iters, std::max<long long>(res->history_capacity, 1));
  CUDA_TRY(ctx->hist.ensure(cap * sizeof(double)));
  CUDA_TRY(ctx->whist.ensure(cap * sizeof(double)));
  CUDA_TRY(launch_loop_init(ctx->st, cfg->max_iters, dt, cfg->tolerance,
                            cfg->time_horizon > 0.0 ? cfg->time_horizon : 0.0, cap, ctx->hist.d(),
                            ctx->whist.d(), ctx->stream));
  ++ctx->launches;
  StepArgs a = ho_args(g, m, c, dt, galpha, cfg);
  a.st = ctx->st;
  a.buf0 = ctx->v0.d();
  a.buf1 = ctx->v1.d();
  a.stage1 = ctx->v2.d();
  a.stage2 = ctx->v3.d();
  a.loop = 1;
  Stage st[3];
  const int ns = stages_of(cfg->time_order, st);
  if (shape >= 0) {
    h4.tab = m.tab;
    for (int d = 0; d < 4; ++d) {
      h4.off_pos[d] = m.row[d].off_pos;
      h4.off_neg[d] = m.row[d].off_neg;
      h4.off_a[d] = m.row[d].off_a;
      h4.off_b[d] = m.row[d].off_b;
    }
    h4.c = ctx->pcbuf.d();
    h4.buf0 = ctx->v0.d();
    h4.buf1 = ctx->v1.d();
    h4.stage1 = ctx->v2.d();
    h4.stage2 = ctx->v3.d();
    h4.st = ctx->st;
    h4.dt = dt;
    h4.loop = 1;
    CUDA_TRY(ho4d_make_maps(h4));
  }
  // one loop "sweep" = one full RK step (all of its stages)
  SweepLauncher launch = [&](cudaStream_t s, cudaGraphConditionalHandle h, int use) {
    for (int k = 0; k < ns; ++k) {
      if (shape >= 0) {
        Ho4dArgs x = h4;
        x.src_sel = st[k].src;
        x.dst_sel = st[k].dst;
        x.kind = st[k].kind;
        x.final_stage = k == ns - 1;
        x.handle = h;
        x.use_handle = use;
        const cudaError_t e = launch_ho4d(x, shape, s);
        if (e != cudaSuccess) return e;
        continue;
      }
      StepArgs x = a;
      x.src_sel = st[k].src;
      x.dst_sel = st[k].dst;
      x.kind = st[k].kind;
      x.final_stage = k == ns - 1;
      x.handle = h;
      x.use_handle = use;
      const cudaError_t e = launch_ho_stage(x, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  CUDA_TRY(cudaEventRecord(e0, ctx->stream));
  const int body = 4;
  // small 2D grids: every stage of the whole loop in one cluster launch
  const char* s2d = std::getenv("HJB_SMALL2D");
  const bool small2d = shape < 0 && g.nd == 2 && !(s2d && std::strcmp(s2d, "0") == 0) &&
                       !cfg->target && small2d_ho_smem(g, nullptr, nullptr) <= 200 * 1024;
  int rc = HJB_OK;
  if (small2d) {
    StepArgs x = a;
    x.src = ctx->v0.d();
    x.dst = out;
    const cudaError_t e = launch_small2d_ho(x, cfg->time_order < 1 ? 1 : cfg->time_order,
                                            ctx->stream);
    if (e != cudaSuccess) rc = set_err(HJB_ERR_CUDA, std::string("small2d_ho: ") + cudaGetErrorString(e));
  } else {
    rc = run_loop(ctx, launch, body);
  }
  if (rc) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return rc;
  }
  CUDA_TRY(cudaEventRecord(e1, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(LoopState), cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const LoopState& ls = *ctx->st_host;
  ctx->launches += small2d ? 1 : (ls.iter + body) * ns;
  res->kernel = small2d ? HJB_KERNEL_SMALL2D_HO : (shape >= 0 ? HJB_KERNEL_HO4D : HJB_KERNEL_HO_GENERIC);
  res->iterations = ls.iter;
  res->converged = ls.converged;
  res->final_residual = ls.last_residual;
  res->wall_seconds = ms * 1e-3;
  const long long nh = std::min<long long>(ls.iter, res->history_capacity);
  if (nh > 0 && res->residual_history)
    CUDA_TRY(cudaMemcpyAsync(res->residual_history, ctx->hist.p, nh * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
  if (nh > 0 && res->wall_ms_history)
    CUDA_TRY(cudaMemcpyAsync(res->wall_ms_history, ctx->whist.p, nh * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
  const double* fin = (ls.iter & 1) ? ctx->v1.d() : ctx->v0.d();
  if (small2d) {
    // the cluster kernel wrote V* to `out` itself
  } else if (shape >= 0) {
    CUDA_TRY(ho4d_unpad(fin, out, g.n[0], h4, ctx->stream));
    ++ctx->launches;
  } else {
    CUDA_TRY(cudaMemcpyAsync(out, fin, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (ls.status == HJB_ERR_DIVERGED)
    return set_err(HJB_ERR_DIVERGED, "solve: diverging (residual grew 10x above its minimum)");
  return HJB_OK;
}

// One full TVD-RK step (all stages), vi_step semantics for orders > 1.
int ho_vi_step(hjb_context* ctx, const DevGrid& g, const DevModel& m, const double* v,
               const double* c, const hjb_solve_config* cfg, double dt, const double* galpha,
               double* out) {
  if (g.nd > 4) return set_err(HJB_ERR_UNSUPPORTED, "vi_step: high-order schemes up to rank 4");
  const size_t bytes = static_cast<size_t>(g.size) * sizeof(double);
  CUDA_TRY(ctx->v2.ensure(bytes));
  CUDA_TRY(ctx->v3.ensure(bytes));
  CUDA_TRY(ctx->v1.ensure(bytes));
  StepArgs a = ho_args(g, m, c, dt, galpha, cfg);
  a.st = ctx->st;
  a.loop = 0;
  a.src = v;
  a.dst = (out == v) ? ctx->v1.d() : out;
  a.stage1 = ctx->v2.d();
  a.stage2 = ctx->v3.d();
  CUDA_TRY(cudaMemsetAsync(ctx->st, 0, sizeof(LoopState), ctx->stream));
  Stage st[3];
  const int ns = stages_of(cfg->time_order, st);
  for (int k = 0; k < ns; ++k) {
    StepArgs x = a;
    x.src_sel = st[k].src;
    x.dst_sel = st[k].dst;
    x.kind = st[k].kind;
    x.final_stage = 0;
    CUDA_TRY(launch_ho_stage(x, ctx->stream));
    ++ctx->launches;
  }
  if (a.dst != out)
    CUDA_TRY(cudaMemcpyAsync(out, a.dst, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return HJB_OK;
}

}  // namespace hjb
