// hjb_shard.cu — multi-GPU slab partition of the 4D solve.
//
// One process per GPU.  Axis 0 (the slowest, so slabs are contiguous) is
// split into balanced slabs; every rank keeps its slab plus one halo plane
// per interior side in the padded layout of k_fast4d.  Per sweep:
//   1. halo exchange of the first/last owned planes with the neighbours
//      (ncclSend/ncclRecv in one group);
//   2. k_fast4d over the owned planes (loop mode 2: halo planes are read as
//      neighbours, the global edges keep the reference's zero ghost rule);
//   3. ncclAllReduce(max) of the sweep's max|dV| bits (non-negative doubles
//      order like uint64);
//   4. k_epilogue: the solve() loop logic on the global max, identical on
//      every rank, so all ranks stop at the same sweep.
// The whole loop is one CUDA graph with a WHILE node; the body holds an even
// number of sweeps with fixed buffers (NCCL needs fixed pointers), which the
// parity of the loop state matches because the loop starts at iteration 0.
// A Jacobi sweep reads only the previous iterate, so the slab result is
// bitwise identical to the single-GPU solve.
//
// NCCL is loaded with dlopen at communicator creation, so libhjb.so carries
// no hard dependency on it (single-GPU use never loads it).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstdlib>
#include <functional>
#include <cstring>
#include <string>

#include "../../include/hjb.h"
#include "hjb_common.cuh"
#include "hjb_fast4d.cuh"
#include "hjb_internal.cuh"
#include "hjb_kernels.cuh"

namespace hjb {
namespace {

// minimal NCCL ABI (nccl.h 2.x)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclUint64_ = 5, ncclFloat64_ = 8 };
enum { ncclMax_ = 2 };

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) =
      nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl* nccl() {
  static Nccl api;
  static bool tried = false;
  if (tried) return api.h ? &api : nullptr;
  tried = true;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h) return nullptr;
#define SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f))
  SYM(GetUniqueId);
  SYM(CommInitRank);
  SYM(CommDestroy);
  SYM(GroupStart);
  SYM(GroupEnd);
  SYM(Send);
  SYM(Recv);
  SYM(AllReduce);
  SYM(GetErrorString);
#undef SYM
  if (!api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllReduce) {
    api.h = nullptr;
    return nullptr;
  }
  return &api;
}

#define NCCL_TRY(expr)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (expr);                                                            \
    if (r_ != 0)                                                                         \
      return set_err(HJB_ERR_NCCL, std::string(#expr " failed: ") +                      \
                                       (nccl()->GetErrorString ? nccl()->GetErrorString(r_) \
                                                               : "nccl error"));         \
  } while (0)

}  // namespace
}  // namespace hjb

struct hjb_comm {
  hjb::ncclComm_t comm = nullptr;
  int nranks = 1;
  int rank = 0;
};

using namespace hjb;

namespace hjb {
namespace {

// WHILE-conditional graph whose body is `body` calls of iter(k, handle, 1)
// (k = position in the body), or the host-polled loop under HJB_LOOP=poll.
int run_sharded_loop(hjb_context* ctx, int body,
                     const std::function<int(int, cudaGraphConditionalHandle, int)>& iter) {
  int rc = HJB_OK;
  const char* mode = std::getenv("HJB_LOOP");
  if (mode && std::strcmp(mode, "poll") == 0) {
    for (;;) {
      for (int k = 0; k < body; ++k)
        if ((rc = iter(k, 0, 0))) return rc;
      CUDA_TRY(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(LoopState), cudaMemcpyDeviceToHost,
                               ctx->stream));
      CUDA_TRY(cudaStreamSynchronize(ctx->stream));
      if (ctx->st_host->done) break;
    }
    return HJB_OK;
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  CUDA_TRY(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle handle;
  do {
    cudaError_t e = cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault);
    if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, graph, nullptr, 0, &cp);
    if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
    e = cudaStreamBeginCaptureToGraph(ctx->stream, cp.conditional.phGraph_out[0], nullptr,
                                      nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
    for (int k = 0; k < body && rc == HJB_OK; ++k) rc = iter(k, handle, 1);
    cudaGraph_t captured = nullptr;
    e = cudaStreamEndCapture(ctx->stream, &captured);
    if (rc) break;
    if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
    e = cudaGraphInstantiate(&exec, graph, 0);
    if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
    e = cudaGraphLaunch(exec, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
  } while (0);
  if (exec) cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  return rc;
}

// stage table of a TVD-RK step: (input, output, kind); buffers 0 = V_n
// (parity), 1 = stage1, 2 = stage2
struct HoStage {
  int src, dst, kind;
};
int ho_stages(int rk, HoStage* st) {
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

// ENO/TVD-RK slab solve: halo of R = order planes per interior side,
// exchanged before every stage, k_ho4t/k_ho4d over the owned
// planes, all-reduce(max) + epilogue after the last stage of a step.
int solve_sharded_ho(hjb_context* ctx, hjb_comm* comm, Nccl* api, const Prepared& p,
                     const hjb_solve_config* cfg, double dt, const double* galpha,
                     uint32_t owned, bool has_lo, bool has_hi, const double* init_slab,
                     const double* c_slab, double* value_slab_out, hjb_solve_result* res) {
  const int r = comm->rank;
  const uint32_t R = cfg->spatial_order < 1 ? 1u : (uint32_t)cfg->spatial_order;
  if ((has_lo || has_hi) && owned < R)
    return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: slab thinner than the ENO halo");
  const uint32_t nloc = owned + (has_lo ? R : 0) + (has_hi ? R : 0);
  DevGrid gloc = p.g;
  gloc.n[0] = nloc;
  Ho4dArgs h;
  std::memset(&h, 0, sizeof h);
  h.order = (int)(R > 3 ? 3 : R);
  h.cbeg = has_lo ? R : 0u;
  h.cend = h.cbeg + owned;
  // Lax-Friedrichs: the global alphas come from the all-reduced scan
  fill_lf(p.hm.dm, scheme_of(cfg), galpha, h.lf, h.lp);
  ho4d_config(gloc, sm_count(ctx->device), h);
  if (h.lf && !h.tma)
    return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: Lax-Friedrichs high order needs the TMA kernels");
  const uint64_t plane = ho4d_plane(h);  // stage-buffer plane (ghost layout of h)
  const size_t lbytes = static_cast<size_t>(nloc) * plane * sizeof(double);
  DevBuf* bufs[4] = {&ctx->v0, &ctx->v1, &ctx->v2, &ctx->v3};
  for (DevBuf* b : bufs) {
    CUDA_TRY(b->ensure(lbytes));
    CUDA_TRY(cudaMemsetAsync(b->p, 0, lbytes, ctx->stream));
  }
  CUDA_TRY(ctx->pcbuf.ensure(lbytes));
  CUDA_TRY(cudaMemsetAsync(ctx->pcbuf.p, 0, lbytes, ctx->stream));
  CUDA_TRY(ho4d_pad(init_slab, ctx->v0.d() + h.cbeg * plane, owned, h, ctx->stream));
  CUDA_TRY(ho4d_pad(c_slab, ctx->pcbuf.d() + h.cbeg * plane, owned, h, ctx->stream));
  ctx->launches += 2;
  h.tab = p.hm.dm.tab;
  for (int d = 0; d < 4; ++d) {
    h.off_pos[d] = p.hm.dm.row[d].off_pos;
    h.off_neg[d] = p.hm.dm.row[d].off_neg;
    h.off_a[d] = p.hm.dm.row[d].off_a;
    h.off_b[d] = p.hm.dm.row[d].off_b;
  }
  h.c = ctx->pcbuf.d();
  h.buf0 = ctx->v0.d();
  h.buf1 = ctx->v1.d();
  h.stage1 = ctx->v2.d();
  h.stage2 = ctx->v3.d();
  h.st = ctx->st;
  h.dt = dt;
  h.loop = 2;
  CUDA_TRY(ho4d_make_maps(h));
  const long long cap =
      std::min<long long>(cfg->max_iters, std::max<long long>(res->history_capacity, 1));
  CUDA_TRY(ctx->hist.ensure(cap * sizeof(double)));
  CUDA_TRY(ctx->whist.ensure(cap * sizeof(double)));
  CUDA_TRY(launch_loop_init(ctx->st, cfg->max_iters, dt, cfg->tolerance,
                            cfg->time_horizon > 0.0 ? cfg->time_horizon : 0.0, cap,
                            ctx->hist.d(), ctx->whist.d(), ctx->stream));
  ++ctx->launches;
  HoStage stages[3];
  const int ns = ho_stages(cfg->time_order, stages);
  unsigned long long* maxbits = &ctx->st->maxdv_bits;
  const size_t pe = static_cast<size_t>(plane);
  auto step = [&](int k, cudaGraphConditionalHandle hd, int use) -> int {
    for (int q = 0; q < ns; ++q) {
      double* src = stages[q].src == 0 ? ((k & 1) ? h.buf1 : h.buf0)
                                       : (stages[q].src == 1 ? h.stage1 : h.stage2);
      if (comm->nranks > 1) {
        NCCL_TRY(api->GroupStart());
        if (has_lo) {
          NCCL_TRY(api->Send(src + h.cbeg * pe, R * pe, ncclFloat64_, r - 1, comm->comm,
                             ctx->stream));
          NCCL_TRY(api->Recv(src + (h.cbeg - R) * pe, R * pe, ncclFloat64_, r - 1, comm->comm,
                             ctx->stream));
        }
        if (has_hi) {
          NCCL_TRY(api->Send(src + (h.cend - R) * pe, R * pe, ncclFloat64_, r + 1, comm->comm,
                             ctx->stream));
          NCCL_TRY(api->Recv(src + h.cend * pe, R * pe, ncclFloat64_, r + 1, comm->comm,
                             ctx->stream));
        }
        NCCL_TRY(api->GroupEnd());
      }
      Ho4dArgs x = h;
      x.src_sel = stages[q].src;
      x.dst_sel = stages[q].dst;
      x.kind = stages[q].kind;
      x.final_stage = q == ns - 1;
      CUDA_TRY(launch_ho4d(x, p.shape, ctx->stream));
    }
    NCCL_TRY(api->AllReduce(maxbits, maxbits, 1, ncclUint64_, ncclMax_, comm->comm, ctx->stream));
    CUDA_TRY(launch_epilogue(ctx->st, hd, use, ctx->stream));
    return HJB_OK;
  };
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  CUDA_TRY(cudaEventRecord(e0, ctx->stream));
  int rc = run_sharded_loop(ctx, 2, step);  // even body: parity of position k == iteration
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
  const LoopState& st = *ctx->st_host;
  ctx->launches += (ns + 1) * (st.iter + 2);
  res->iterations = st.iter;
  res->converged = st.converged;
  res->final_residual = st.last_residual;
  res->wall_seconds = ms * 1e-3;
  const long long nh = std::min<long long>(st.iter, res->history_capacity);
  if (nh > 0 && res->residual_history)
    CUDA_TRY(cudaMemcpyAsync(res->residual_history, ctx->hist.p, nh * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
  if (nh > 0 && res->wall_ms_history)
    CUDA_TRY(cudaMemcpyAsync(res->wall_ms_history, ctx->whist.p, nh * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
  const double* fin = ((st.iter & 1) ? h.buf1 : h.buf0) + h.cbeg * pe;
  CUDA_TRY(ho4d_unpad(fin, value_slab_out, owned, h, ctx->stream));
  ++ctx->launches;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (st.status == HJB_ERR_DIVERGED)
    return set_err(HJB_ERR_DIVERGED, "solve: diverging (residual grew 10x above its minimum)");
  return HJB_OK;
}

}  // namespace
}  // namespace hjb

extern "C" {

int hjb_slab_partition(int64_t n0, int32_t nranks, int32_t rank, int64_t* begin, int64_t* end) {
  if (nranks < 1 || rank < 0 || rank >= nranks || n0 < nranks)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "slab_partition: need 0 <= rank < nranks <= n0");
  const int64_t base = n0 / nranks, extra = n0 % nranks;
  *begin = rank * base + (rank < extra ? rank : extra);
  *end = *begin + base + (rank < extra ? 1 : 0);
  return HJB_OK;
}

int hjb_nccl_unique_id(void* out) {
  Nccl* api = nccl();
  if (!api) return set_err(HJB_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  NCCL_TRY(api->GetUniqueId(&id));
  std::memcpy(out, &id, sizeof id);
  return HJB_OK;
}

int hjb_comm_create(hjb_context* ctx, int32_t nranks, int32_t rank, const void* unique_id,
                    hjb_comm** out) {
  if (!ctx || !out || !unique_id) return set_err(HJB_ERR_INVALID_ARGUMENT, "comm_create: null");
  Nccl* api = nccl();
  if (!api) return set_err(HJB_ERR_NCCL, "libnccl.so.2 not loadable");
  CUDA_TRY(cudaSetDevice(ctx->device));
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof id);
  hjb_comm* c = new hjb_comm();
  c->nranks = nranks;
  c->rank = rank;
  const ncclResult_t r = api->CommInitRank(&c->comm, nranks, id, rank);
  if (r != 0) {
    delete c;
    return set_err(HJB_ERR_NCCL, std::string("ncclCommInitRank failed: ") +
                                     (api->GetErrorString ? api->GetErrorString(r) : ""));
  }
  *out = c;
  return HJB_OK;
}

int hjb_comm_destroy(hjb_comm* c) {
  if (!c) return HJB_OK;
  if (c->comm && nccl() && nccl()->CommDestroy) nccl()->CommDestroy(c->comm);
  delete c;
  return HJB_OK;
}

// One sweep over planes [plane_begin, plane_end) of a full 4D grid (device
// pointers, reference layout): the slab computation of rank r on one device.
// Writes only those planes of `out` and the slab's max|dV| to *max_dv.
int hjb_sweep_planes_dev(hjb_context* ctx, const hjb_grid* gi, const hjb_model* mi,
                         const hjb_dbounds* db, const double* value, const double* constraint,
                         int64_t plane_begin, int64_t plane_end, double dt, double* out,
                         double* max_dv) {
  int rc;
  if (!ctx) return set_err(HJB_ERR_INVALID_ARGUMENT, "context: null");
  CUDA_TRY(cudaSetDevice(ctx->device));
  Prepared p;
  if ((rc = prepare(ctx, gi, mi, db, p))) return rc;
  if (p.shape < 0)
    return set_err(HJB_ERR_UNSUPPORTED, "sweep_planes: model/grid outside the 4D fast path");
  if (plane_begin < 0 || plane_end > p.g.n[0] || plane_begin >= plane_end)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "sweep_planes: bad plane range");
  Fast4dArgs f;
  std::memset(&f, 0, sizeof f);
  f.kcells = 2;
  f.maxthreads = 576;
  f.cbeg = static_cast<uint32_t>(plane_begin);
  f.cend = static_cast<uint32_t>(plane_end);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  f.tab_len = static_cast<uint32_t>(p.hm.tab.size());
  fast4d_config(p.g, sms > 0 ? sms : 148, f);
  const uint64_t rows = static_cast<uint64_t>(p.g.n[0]) * p.g.n[1] * p.g.n[2];
  const size_t pb = rows * f.n3p * sizeof(double);
  DevBuf a, bbuf, cb;
  CUDA_TRY(a.ensure(pb));
  CUDA_TRY(bbuf.ensure(pb));
  CUDA_TRY(cb.ensure(pb));
  CUDA_TRY(launch_pad4(value, a.d(), rows, p.g.n[3], f.n3p, ctx->stream));
  CUDA_TRY(launch_pad4(constraint, cb.d(), rows, p.g.n[3], f.n3p, ctx->stream));
  CUDA_TRY(launch_pad4(value, bbuf.d(), rows, p.g.n[3], f.n3p, ctx->stream));
  fill_tables(p, f);
  f.c = cb.d();
  f.buf0 = a.d();
  f.buf1 = bbuf.d();
  f.src = a.d();
  f.dst = bbuf.d();
  CUDA_TRY(fast4d_make_maps(f, a.d(), bbuf.d(), cb.d()));
  f.st = ctx->st;
  f.dt = dt;
  f.loop = 0;
  CUDA_TRY(cudaMemsetAsync(ctx->st, 0, sizeof(LoopState), ctx->stream));
  CUDA_TRY(launch_fast4d(f, p.shape, ctx->stream));
  CUDA_TRY(launch_unpad4(bbuf.d(), out, rows, p.g.n[3], f.n3p, ctx->stream));
  ctx->launches += 5;
  unsigned long long bits = 0;
  CUDA_TRY(cudaMemcpyAsync(&bits, &ctx->st->maxdv_bits, sizeof bits, cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  std::memcpy(max_dv, &bits, sizeof bits);
  return HJB_OK;
}

int hjb_ho_stage_planes_dev(hjb_context* ctx, const hjb_grid* gi, const hjb_model* mi,
                            const hjb_dbounds* db, const double* stage_in, const double* value_n,
                            const double* constraint, double dt, int32_t order, int32_t kind,
                            int64_t plane_begin, int64_t plane_end, double* out,
                            double* max_dv) {
  int rc;
  if (!ctx) return set_err(HJB_ERR_INVALID_ARGUMENT, "context: null");
  CUDA_TRY(cudaSetDevice(ctx->device));
  Prepared p;
  if ((rc = prepare(ctx, gi, mi, db, p))) return rc;
  if (p.shape < 0)
    return set_err(HJB_ERR_UNSUPPORTED, "ho_stage_planes: model/grid outside the 4D fast path");
  if (plane_begin < 0 || plane_end > p.g.n[0] || plane_begin >= plane_end)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "ho_stage_planes: bad plane range");
  if (order < 1 || order > 3 || kind < 0 || kind > 3)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "ho_stage_planes: bad order/kind");
  Ho4dArgs h;
  std::memset(&h, 0, sizeof h);
  h.order = order;
  h.cbeg = static_cast<uint32_t>(plane_begin);
  h.cend = static_cast<uint32_t>(plane_end);
  ho4d_config(p.g, sm_count(ctx->device), h);
  const uint32_t n0 = p.g.n[0];
  const size_t pb = n0 * ho4d_plane(h) * sizeof(double);
  DevBuf a, vn, cb, o;
  CUDA_TRY(a.ensure(pb));
  CUDA_TRY(vn.ensure(pb));
  CUDA_TRY(cb.ensure(pb));
  CUDA_TRY(o.ensure(pb));
  CUDA_TRY(ho4d_pad(stage_in, a.d(), n0, h, ctx->stream));
  CUDA_TRY(ho4d_pad(value_n, vn.d(), n0, h, ctx->stream));
  CUDA_TRY(ho4d_pad(constraint, cb.d(), n0, h, ctx->stream));
  CUDA_TRY(ho4d_pad(stage_in, o.d(), n0, h, ctx->stream));
  h.tab = p.hm.dm.tab;
  for (int d = 0; d < 4; ++d) {
    h.off_pos[d] = p.hm.dm.row[d].off_pos;
    h.off_neg[d] = p.hm.dm.row[d].off_neg;
    h.off_a[d] = p.hm.dm.row[d].off_a;
    h.off_b[d] = p.hm.dm.row[d].off_b;
  }
  h.c = cb.d();
  h.xsrc = a.d();
  h.xvn = vn.d();
  h.xdst = o.d();
  h.kind = kind;
  h.final_stage = 1;
  h.loop = 0;
  h.st = ctx->st;
  h.dt = dt;
  CUDA_TRY(ho4d_make_maps(h));
  CUDA_TRY(cudaMemsetAsync(ctx->st, 0, sizeof(LoopState), ctx->stream));
  CUDA_TRY(launch_ho4d(h, p.shape, ctx->stream));
  CUDA_TRY(ho4d_unpad(o.d(), out, n0, h, ctx->stream));
  ctx->launches += 6;
  unsigned long long bits = 0;
  CUDA_TRY(cudaMemcpyAsync(&bits, &ctx->st->maxdv_bits, sizeof bits, cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  std::memcpy(max_dv, &bits, sizeof bits);
  return HJB_OK;
}

int hjb_solve_sharded_dev(hjb_context* ctx, hjb_comm* comm, const hjb_grid* gi,
                          const hjb_model* mi, const hjb_dbounds* db, const double* init_slab,
                          const double* c_slab, const hjb_solve_config* cfg,
                          double* value_slab_out, hjb_solve_result* res) {
  int rc;
  if (!ctx || !comm) return set_err(HJB_ERR_INVALID_ARGUMENT, "solve_sharded: null context/comm");
  CUDA_TRY(cudaSetDevice(ctx->device));
  if ((rc = validate_config(cfg))) return rc;
  Prepared p;
  if ((rc = prepare(ctx, gi, mi, db, p))) return rc;
  if (p.shape < 0)
    return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: model/grid outside the 4D fast path");
  const bool high_order = cfg->spatial_order > 1 || cfg->time_order > 1;
  // the scheme's own variant of the fast path (first and high order)
  const int scheme = scheme_of(cfg);
  if (fast4d_shape(p.g, p.hm.dm, scheme) != p.shape)
    return set_err(HJB_ERR_UNSUPPORTED,
                   "solve_sharded: Lax-Friedrichs needs one input term per row of the 4D model");
  Nccl* api = nccl();
  if (!api) return set_err(HJB_ERR_NCCL, "libnccl.so.2 not loadable");
  const int P = comm->nranks, r = comm->rank;
  int64_t slab_b, slab_e;
  if ((rc = hjb_slab_partition(p.g.n[0], P, r, &slab_b, &slab_e))) return rc;
  const uint32_t owned = static_cast<uint32_t>(slab_e - slab_b);
  const bool has_lo = r > 0, has_hi = r < P - 1;
  // Every rank must reject a too-thin partition BEFORE the first collective:
  // balanced slabs differ by one plane, so a per-rank check would let the
  // thicker ranks enter NCCL while a thin one returns (a hang, not an error).
  // The smallest slab is floor(n0 / P) planes on every rank's view.
  {
    const int64_t R = high_order ? (cfg->spatial_order < 1 ? 1 : cfg->spatial_order) : 1;
    if (P > 1 && static_cast<int64_t>(p.g.n[0]) / P < R)
      return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: slab thinner than the ENO halo");
  }
  const uint32_t nloc = owned + (has_lo ? 1 : 0) + (has_hi ? 1 : 0);

  // CFL scan over the slab + all-reduce(max): rows of the fast path never
  // depend on x0, so the slab's local grid gives the global values
  DevGrid gl = p.g;
  gl.n[0] = owned;
  gl.size = owned * gl.stride[0];
  gl.divs[0].init(owned);
  Scan s;
  if ((rc = run_scan(ctx, gl, p.hm.dm, s))) return rc;
  {
    unsigned long long bits[1 + kMaxDims];
    std::memcpy(bits, &s.max_speed_sum, sizeof(double));
    std::memcpy(bits + 1, s.max_alpha, kMaxDims * sizeof(double));
    unsigned long long* dbits = reinterpret_cast<unsigned long long*>(ctx->scratch.d());
    CUDA_TRY(cudaMemcpyAsync(dbits, bits, sizeof bits, cudaMemcpyHostToDevice, ctx->stream));
    NCCL_TRY(api->AllReduce(dbits, dbits, 1 + kMaxDims, ncclUint64_, ncclMax_, comm->comm,
                            ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(bits, dbits, sizeof bits, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    std::memcpy(&s.max_speed_sum, bits, sizeof(double));
    std::memcpy(s.max_alpha, bits + 1, kMaxDims * sizeof(double));
  }
  if (!(s.max_speed_sum > 0.0))
    return set_err(HJB_ERR_RUNTIME, "solve: flow is identically zero on the grid");
  const double dt = cfg->cfl_factor / s.max_speed_sum;
  hjb_solve_result local;
  std::memset(&local, 0, sizeof local);
  if (!res) res = &local;
  res->dt = dt;
  res->nodes_per_sweep = p.g.size;
  res->iterations = 0;
  res->converged = 0;
  if (cfg->max_iters == 0) {
    CUDA_TRY(cudaMemcpyAsync(value_slab_out, init_slab,
                             static_cast<size_t>(owned) * p.g.stride[0] * sizeof(double),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return HJB_OK;
  }

  if (high_order)
    return solve_sharded_ho(ctx, comm, api, p, cfg, dt, s.max_alpha, owned, has_lo, has_hi,
                            init_slab, c_slab,
                            value_slab_out, res);

  // local padded slab arrays: [halo_lo?][owned][halo_hi?]
  DevGrid gloc = p.g;
  gloc.n[0] = nloc;
  Fast4dArgs f;
  std::memset(&f, 0, sizeof f);
  f.kcells = 2;
  f.maxthreads = 576;
  f.cbeg = has_lo ? 1u : 0u;
  f.cend = f.cbeg + owned;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  f.tab_len = static_cast<uint32_t>(p.hm.tab.size());
  fast4d_config(gloc, sms > 0 ? sms : 148, f);
  const uint64_t plane = static_cast<uint64_t>(p.g.n[1]) * p.g.n[2] * f.n3p;  // padded plane
  const uint64_t rows_owned = static_cast<uint64_t>(owned) * p.g.n[1] * p.g.n[2];
  const size_t lbytes = static_cast<size_t>(nloc) * plane * sizeof(double);
  CUDA_TRY(ctx->v2.ensure(lbytes));
  CUDA_TRY(ctx->v3.ensure(lbytes));
  CUDA_TRY(ctx->pcbuf.ensure(lbytes));
  CUDA_TRY(cudaMemsetAsync(ctx->v2.p, 0, lbytes, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(ctx->v3.p, 0, lbytes, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(ctx->pcbuf.p, 0, lbytes, ctx->stream));
  double* own0 = ctx->v2.d() + f.cbeg * plane;
  CUDA_TRY(launch_pad4(init_slab, own0, rows_owned, p.g.n[3], f.n3p, ctx->stream));
  CUDA_TRY(launch_pad4(c_slab, ctx->pcbuf.d() + f.cbeg * plane, rows_owned, p.g.n[3], f.n3p,
                       ctx->stream));
  ctx->launches += 2;
  fill_tables(p, f);
  fill_lf(p.hm.dm, scheme, s.max_alpha, f);
  if (f.lf) {  // the Lax-Friedrichs variant's CTA size
    f.maxthreads = 448;
    f.cbeg = has_lo ? 1u : 0u;
    f.cend = f.cbeg + owned;
    fast4d_config(gloc, sms > 0 ? sms : 148, f);
  }
  f.c = ctx->pcbuf.d();
  f.buf0 = ctx->v2.d();
  f.buf1 = ctx->v3.d();
  CUtensorMap map_b0, map_b1;
  CUDA_TRY(fast4d_make_maps(f, f.buf0, f.buf1, f.c));
  map_b0 = f.map0;
  map_b1 = f.map1;
  f.st = ctx->st;
  f.dt = dt;
  f.loop = 2;

  const long long cap =
      std::min<long long>(cfg->max_iters, std::max<long long>(res->history_capacity, 1));
  CUDA_TRY(ctx->hist.ensure(cap * sizeof(double)));
  CUDA_TRY(ctx->whist.ensure(cap * sizeof(double)));
  CUDA_TRY(launch_loop_init(ctx->st, cfg->max_iters, dt, cfg->tolerance,
                            cfg->time_horizon > 0.0 ? cfg->time_horizon : 0.0, cap,
                            ctx->hist.d(), ctx->whist.d(), ctx->stream));
  ++ctx->launches;
  unsigned long long* maxbits = &ctx->st->maxdv_bits;
  const size_t pe = static_cast<size_t>(plane);
  // one sweep at a fixed buffer parity: exchange, sweep, all-reduce, epilogue
  auto sweep = [&](int k, cudaGraphConditionalHandle h, int use) -> int {
    double* src = (k & 1) ? f.buf1 : f.buf0;
    double* dst = (k & 1) ? f.buf0 : f.buf1;
    if (P > 1) {
      NCCL_TRY(api->GroupStart());
      if (has_lo) {
        NCCL_TRY(api->Send(src + f.cbeg * pe, pe, ncclFloat64_, r - 1, comm->comm, ctx->stream));
        NCCL_TRY(api->Recv(src, pe, ncclFloat64_, r - 1, comm->comm, ctx->stream));
      }
      if (has_hi) {
        NCCL_TRY(api->Send(src + (f.cend - 1) * pe, pe, ncclFloat64_, r + 1, comm->comm,
                           ctx->stream));
        NCCL_TRY(api->Recv(src + f.cend * pe, pe, ncclFloat64_, r + 1, comm->comm, ctx->stream));
      }
      NCCL_TRY(api->GroupEnd());
    }
    Fast4dArgs x = f;
    x.src = src;
    x.dst = dst;
    x.map0 = (k & 1) ? map_b1 : map_b0;
    CUDA_TRY(launch_fast4d(x, p.shape, ctx->stream));
    NCCL_TRY(api->AllReduce(maxbits, maxbits, 1, ncclUint64_, ncclMax_, comm->comm, ctx->stream));
    CUDA_TRY(launch_epilogue(ctx->st, h, use, ctx->stream));
    return HJB_OK;
  };
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  CUDA_TRY(cudaEventRecord(e0, ctx->stream));
  const int body = 8;  // even: buffer parity of position k == iteration parity
  const char* mode = std::getenv("HJB_LOOP");
  if (mode && std::strcmp(mode, "poll") == 0) {
    for (;;) {
      for (int k = 0; k < body; ++k)
        if ((rc = sweep(k, 0, 0))) return rc;
      CUDA_TRY(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(LoopState), cudaMemcpyDeviceToHost,
                               ctx->stream));
      CUDA_TRY(cudaStreamSynchronize(ctx->stream));
      if (ctx->st_host->done) break;
    }
  } else {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    CUDA_TRY(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle handle;
    rc = HJB_OK;
    do {
      cudaError_t e = cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault);
      if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = handle;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      e = cudaGraphAddNode(&node, graph, nullptr, 0, &cp);
      if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
      e = cudaStreamBeginCaptureToGraph(ctx->stream, cp.conditional.phGraph_out[0], nullptr,
                                        nullptr, 0, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
      for (int k = 0; k < body && rc == HJB_OK; ++k) rc = sweep(k, handle, 1);
      cudaGraph_t captured = nullptr;
      e = cudaStreamEndCapture(ctx->stream, &captured);
      if (rc) break;
      if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
      e = cudaGraphInstantiate(&exec, graph, 0);
      if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
      e = cudaGraphLaunch(exec, ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) { rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e)); break; }
    } while (0);
    if (exec) cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (rc) return rc;
  }
  CUDA_TRY(cudaEventRecord(e1, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(LoopState), cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const LoopState& st = *ctx->st_host;
  ctx->launches += 2 * (st.iter + body);
  res->iterations = st.iter;
  res->converged = st.converged;
  res->final_residual = st.last_residual;
  res->wall_seconds = ms * 1e-3;
  const long long nh = std::min<long long>(st.iter, res->history_capacity);
  if (nh > 0 && res->residual_history)
    CUDA_TRY(cudaMemcpyAsync(res->residual_history, ctx->hist.p, nh * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
  if (nh > 0 && res->wall_ms_history)
    CUDA_TRY(cudaMemcpyAsync(res->wall_ms_history, ctx->whist.p, nh * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
  const double* fin = ((st.iter & 1) ? f.buf1 : f.buf0) + f.cbeg * pe;
  CUDA_TRY(launch_unpad4(fin, value_slab_out, rows_owned, p.g.n[3], f.n3p, ctx->stream));
  ++ctx->launches;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (st.status == HJB_ERR_DIVERGED)
    return set_err(HJB_ERR_DIVERGED, "solve: diverging (residual grew 10x above its minimum)");
  return HJB_OK;
}

}  // extern "C"
