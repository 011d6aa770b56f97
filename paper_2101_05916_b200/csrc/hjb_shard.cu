// hjb_shard.cu — multi-GPU slab partition of the 4D solve.
//
// One process per GPU.  Axis 0 (the slowest, so slabs are contiguous) is
// split into balanced slabs; every rank keeps its slab plus R halo planes
// per interior side (R = 1 first order, the ENO order otherwise) in the
// padded / ghost layout of the 4D kernels.  Per loop position and RK stage:
//   1. the BOUNDARY planes (the R owned planes next to each neighbour — what
//      the neighbours read next) are swept first (one launch over both
//      ranges, Fast4dArgs/Ho4dArgs split ranges);
//   2. on a second captured stream, the stage output's boundary planes go to
//      the neighbours' halo planes (grouped ncclSend/ncclRecv) while
//   3. the INTERIOR planes sweep on the main stream (they never read halos);
//   4. join; after the last stage ncclAllReduce(max) of the max|dV| bits
//      (non-negative doubles order like uint64) and k_epilogue run the
//      solve() loop logic on the global max, identically on every rank, so
//      all ranks leave the device loop together.
// The whole loop is one CUDA graph with a WHILE node; the body holds an even
// number of positions with fixed buffers (NCCL needs fixed pointers), which
// the parity of the loop state matches because the loop starts at 0.  A
// Jacobi sweep / RK stage reads only the previous stage, so the slab result
// is bitwise identical to the single-GPU solve.
//
// hjb_solve_sharded_local_dev runs the SAME per-rank plans (geometry, halo
// offsets, boundary/interior launches, epilogues) for P in-process ranks on
// one device, with the halo planes moved by device copies on the second
// stream and the all-reduce by a kernel: the multi-rank protocol exercised
// and timed on a single GPU (no kernel waits on another).
//
// NCCL is loaded with dlopen at communicator creation, so libhjb.so carries
// no hard dependency on it (single-GPU use never loads it).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <thread>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

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
  hjb::ncclComm_t comm = nullptr;  // null: a peer-store-only communicator (no NCCL)
  int nranks = 1;
  int rank = 0;
  // peer-store transport (HJB_SHARD_P2P): this rank's control block — two
  // halo-epoch flags (written by the lower / upper neighbour over NVLink) at
  // offset 0 and the residual mailbox (P2PMbox) at kMboxOffset — plus the
  // epoch counters, all monotonic across solves so no reset can race a
  // neighbour's write; every rank's control block mapped over CUDA IPC
  // (peer_ctl[q], opened once, closed at destroy)
  unsigned int* p2p_flags = nullptr;
  unsigned int p2p_seq = 0, res_seq = 0, scan_seq = 0, blob_seq = 0;
  std::vector<void*> peer_ctl;
  bool peers_open = false;
};
// control-block layout: halo-epoch flags (2 x u32) | blob epoch (u32) |
// residual mailbox | scan mailbox | the per-solve buffer-handle blob
constexpr size_t kCtlBytes = 4096, kBlobFlagOffset = 64, kMboxOffset = 256, kScanOffset = 512,
                 kBlobOffset = 1024;

using namespace hjb;

namespace hjb {
namespace {

// WHILE-conditional graph whose body is `body` calls of iter(k, handle, 1)
// (k = position in the body), or the host-polled loop under HJB_LOOP=poll
// (loop state of ctx->st).  iter may fork work onto other streams with
// events; they must join back before it returns.
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

// Host-driven loop for the NCCL transport: the positions are issued eagerly
// (no graph capture: NCCL's own stream dependencies stay the eager ones it is
// built for — a captured all-reduce inside the conditional graph, with the
// sweep kernels on a second captured stream, hung on the B200 pool).  Batch j
// (= `body` positions) is followed by an async copy of the loop state's done
// flag; the host waits for batch j - 1's flag only after issuing batch j, so
// the GPU never idles on the host, and every rank stops after the same batch
// (done is identical on all ranks at the same iteration), issuing the same
// NCCL calls.  The extra batch finds done set: its kernels and epilogues
// return at once.
int run_eager_loop(hjb_context* ctx, int body,
                   const std::function<int(int, cudaGraphConditionalHandle, int)>& iter) {
  int* flags = nullptr;  // pinned: done flag after batch j in flags[j & 1]
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int rc = HJB_OK;
  cudaError_t e = cudaMallocHost(&flags, 2 * sizeof(int));
  for (int i = 0; i < 2 && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  if (e != cudaSuccess) rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e));
  for (long long j = 0; rc == HJB_OK; ++j) {
    for (int k = 0; k < body && rc == HJB_OK; ++k) rc = iter(k, 0, 0);
    if (rc) break;
    e = cudaMemcpyAsync(flags + (j & 1), &ctx->st->done, sizeof(int), cudaMemcpyDeviceToHost,
                        ctx->stream);
    if (e == cudaSuccess) e = cudaEventRecord(ev[j & 1], ctx->stream);
    if (e == cudaSuccess && j >= 1) e = cudaEventSynchronize(ev[(j - 1) & 1]);
    if (e != cudaSuccess) {
      rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e));
      break;
    }
    if (j >= 1 && flags[(j - 1) & 1]) break;
  }
  e = cudaStreamSynchronize(ctx->stream);
  if (rc == HJB_OK && e != cudaSuccess) rc = set_err(HJB_ERR_CUDA, cudaGetErrorString(e));
  for (cudaEvent_t x : ev)
    if (x) cudaEventDestroy(x);
  if (flags) cudaFreeHost(flags);
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

// ---------------------------------------------------------------- geometry
// One rank's slab in its local buffers: [halo_lo R][owned][halo_hi R]
// planes (halo planes only next to a neighbour).
struct SlabGeom {
  int P = 1, r = 0;
  uint32_t owned = 0, R = 1, nloc = 0, cbeg = 0, cend = 0;
  int64_t gbeg = 0;  // first owned plane in the global grid
  bool has_lo = false, has_hi = false;
};

SlabGeom slab_geom(uint32_t n0, int P, int r, uint32_t R) {
  SlabGeom s;
  int64_t b = 0, e = 0;
  hjb_slab_partition(n0, P, r, &b, &e);
  s.P = P;
  s.r = r;
  s.R = R;
  s.gbeg = b;
  s.owned = static_cast<uint32_t>(e - b);
  s.has_lo = r > 0;
  s.has_hi = r < P - 1;
  s.cbeg = s.has_lo ? R : 0u;
  s.cend = s.cbeg + s.owned;
  s.nloc = s.owned + (s.has_lo ? R : 0u) + (s.has_hi ? R : 0u);
  return s;
}

// The halo protocol of one stage buffer, in local planes: the first / last
// R owned planes go to the lower / upper neighbour, whose halo planes
// [cbeg - R, cbeg) / [cend, cend + R) receive them.  Both transports (NCCL
// send/recv between processes, device copies between in-process ranks) move
// exactly these planes.
struct Halo {
  uint32_t send_lo, recv_lo, send_hi, recv_hi, planes;
};
Halo halo_of(const SlabGeom& s) {
  return {s.cbeg, s.has_lo ? s.cbeg - s.R : 0u, s.cend - s.R, s.cend, s.R};
}

// Boundary planes (the R owned planes next to each neighbour: what the
// neighbours read next stage) are swept first, so their transfer overlaps
// the sweep of the interior planes.
struct PlaneSplit {
  uint32_t b0 = 0, e0 = 0, b1 = 0, e1 = 0;  // boundary ranges ([b1, e1) may be empty)
  uint32_t i0 = 0, i1 = 0;                  // interior
  bool bnd = false, inner = false;
};
PlaneSplit plane_split(const SlabGeom& s) {
  PlaneSplit x;
  // HJB_SHARD_SPLIT=0 (diagnostic, with HJB_SHARD_OVERLAP=0): one launch
  // over the whole slab, then the exchange
  const char* e = std::getenv("HJB_SHARD_SPLIT");
  if (s.P == 1 || (e && std::strcmp(e, "0") == 0)) {
    x.i0 = s.cbeg;
    x.i1 = s.cend;
    x.inner = true;
    return x;
  }
  const uint32_t lo_end = s.has_lo ? s.cbeg + s.R : s.cbeg;
  const uint32_t hi_beg = s.has_hi ? s.cend - s.R : s.cend;
  x.bnd = true;
  if (lo_end >= hi_beg) {  // the boundary covers the whole slab
    x.b0 = s.cbeg;
    x.e0 = s.cend;
    return x;
  }
  if (s.has_lo) {
    x.b0 = s.cbeg;
    x.e0 = lo_end;
    if (s.has_hi) {
      x.b1 = hi_beg;
      x.e1 = s.cend;
    }
  } else {
    x.b0 = hi_beg;
    x.e0 = s.cend;
  }
  x.i0 = lo_end;
  x.i1 = hi_beg;
  x.inner = true;
  return x;
}

// ------------------------------------------------------------- one rank
enum LaunchMode { kBnd = 0, kInner = 1, kBoth = 2 };
struct SlabRank {
  SlabGeom geo;
  PlaneSplit sp;
  int shape = -1;
  bool ho = false;
  size_t pe = 0;  // elements per local plane
  // launches (first order f*, high order h*): boundary planes only,
  // interior only, and both in one launch with the boundary items first and
  // the completion signal (bnd_flag) for the transfer stream
  Fast4dArgs fb, fi, fc;
  // peer-store halos (first order, HJB_SHARD_P2P): the neighbours' V
  // buffers (by buffer index 0 / 1), the plane of theirs that receives our
  // first send plane, their flag we publish to, our flags they publish to,
  // and the epoch the next launch publishes
  struct P2PLink {
    bool on = false;
    double* peer_buf[2][4] = {};  // [side][buffer: V parity 0 / 1, stage1, stage2]
    uint32_t dst0[2] = {0u, 0u};
    unsigned int* peer_flag[2] = {nullptr, nullptr};
    unsigned int* own_flag[2] = {nullptr, nullptr};
    unsigned int epoch = 0;
  } p2p;
  CUtensorMap map_b0, map_b1;
  Ho4dArgs hb, hi, hc;
  HoStage stages[3];
  int ns = 1;
  double* buf[4] = {nullptr, nullptr, nullptr, nullptr};  // V parity 0/1, stage1, stage2
  LoopState* st = nullptr;

  // the buffer stage q writes at loop position k (its halo travels after it)
  double* stage_out(int k, int q) const {
    const int d = ho ? stages[q].dst : 0;
    if (d == 0) return (k & 1) ? buf[0] : buf[1];
    return d == 1 ? buf[2] : buf[3];
  }
  // V after `iters` completed iterations
  double* value(long long iters) const { return (iters & 1) ? buf[1] : buf[0]; }
  // mode: kBnd / kInner / kBoth; slot: the max|dV| accumulator of
  // position k (null: st->maxdv_bits)
  cudaError_t launch(int k, int q, int mode, unsigned long long* slot, cudaStream_t s) const;
};

cudaError_t SlabRank::launch(int k, int q, int mode, unsigned long long* slot,
                             cudaStream_t s) const {
  if (!ho) {
    Fast4dArgs x = mode == kBnd ? fb : (mode == kInner ? fi : fc);
    x.src = (k & 1) ? buf[1] : buf[0];
    x.dst = (k & 1) ? buf[0] : buf[1];
    x.map0 = (k & 1) ? map_b1 : map_b0;
    x.mdv = slot;
    if (p2p.on && mode == kBoth) {  // boundary planes also into the neighbours' halos
      const Halo h = halo_of(geo);
      const int ob = (k & 1) ? 0 : 1;  // the output buffer index (theirs is the same)
      x.p2p_R = h.planes;
      x.p2p_epoch = p2p.epoch;
      for (int sd = 0; sd < 2; ++sd) {
        x.p2p_dst[sd] = p2p.peer_buf[sd][ob];
        x.p2p_flag[sd] = p2p.peer_flag[sd];
        x.p2p_dst0[sd] = p2p.dst0[sd];
      }
      x.p2p_src0[0] = h.send_lo;
      x.p2p_src0[1] = h.send_hi;
    }
    return launch_fast4d(x, shape, s);
  }
  Ho4dArgs x = mode == kBnd ? hb : (mode == kInner ? hi : hc);
  x.mdv = slot;
  if (p2p.on && mode == kBoth) {  // stage output's boundary planes into the neighbours
    const Halo h = halo_of(geo);
    const int d = stages[q].dst;
    const int ob = d == 0 ? ((k & 1) ? 0 : 1) : (d == 1 ? 2 : 3);
    x.p2p_R = h.planes;
    x.p2p_epoch = p2p.epoch;
    for (int sd = 0; sd < 2; ++sd) {
      x.p2p_dst[sd] = p2p.peer_buf[sd][ob];
      x.p2p_flag[sd] = p2p.peer_flag[sd];
      x.p2p_dst0[sd] = p2p.dst0[sd];
    }
    x.p2p_src0[0] = h.send_lo;
    x.p2p_src0[1] = h.send_hi;
  }
  x.pmode = 1;  // position parity == iteration parity (even body, loop from 0)
  x.parity = k & 1;
  x.src_sel = stages[q].src;
  x.dst_sel = stages[q].dst;
  x.kind = stages[q].kind;
  x.final_stage = q == ns - 1;
  return launch_ho4d(x, shape, s);
}

// Local buffers, padded inputs, launch arguments of one rank.  bufs[0..3] /
// cbuf are grown to the slab's size; init_slab / c_slab hold the owned
// planes (reference layout, device).
int setup_rank(int device, const Prepared& p, const hjb_solve_config* cfg, double dt,
               const double* galpha, const SlabGeom& geo, DevBuf* const bufs[4], DevBuf* cbuf,
               LoopState* st, const double* init_slab, const double* c_slab, cudaStream_t s,
               SlabRank& rk, long long* launches) {
  const int sms = sm_count(device);
  const int scheme = scheme_of(cfg);
  rk.geo = geo;
  rk.sp = plane_split(geo);
  rk.shape = p.shape;
  rk.st = st;
  rk.ho = cfg->spatial_order > 1 || cfg->time_order > 1;
  DevGrid gloc = p.g;
  gloc.n[0] = geo.nloc;
  if (!rk.ho) {
    Fast4dArgs f;
    std::memset(&f, 0, sizeof f);
    f.kcells = 2;
    f.maxthreads = 576;
    f.cbeg = geo.cbeg;
    f.cend = geo.cend;
    f.tab_len = static_cast<uint32_t>(p.hm.tab.size());
    fast4d_config(gloc, sms, f);
    fill_tables(p, f);
    fill_lf(p.hm.dm, scheme, galpha, f);
    if (f.lf) {  // the Lax-Friedrichs variant's CTA size
      f.maxthreads = p.shape == kShapeGen ? 384u : 448u;
      f.cbeg = geo.cbeg;
      f.cend = geo.cend;
      fast4d_config(gloc, sms, f);
    }
    rk.pe = static_cast<size_t>(p.g.n[1]) * p.g.n[2] * f.n3p;
    const uint64_t rows_owned = static_cast<uint64_t>(geo.owned) * p.g.n[1] * p.g.n[2];
    const size_t lbytes = static_cast<size_t>(geo.nloc) * rk.pe * sizeof(double);
    for (int b = 0; b < 2; ++b) {
      CUDA_TRY(bufs[b]->ensure(lbytes));
      CUDA_TRY(cudaMemsetAsync(bufs[b]->p, 0, lbytes, s));
      rk.buf[b] = bufs[b]->d();
    }
    CUDA_TRY(cbuf->ensure(lbytes));
    CUDA_TRY(cudaMemsetAsync(cbuf->p, 0, lbytes, s));
    CUDA_TRY(launch_pad4(init_slab, rk.buf[0] + geo.cbeg * rk.pe, rows_owned, p.g.n[3], f.n3p, s));
    CUDA_TRY(launch_pad4(c_slab, cbuf->d() + geo.cbeg * rk.pe, rows_owned, p.g.n[3], f.n3p, s));
    *launches += 2;
    f.c = cbuf->d();
    f.buf0 = rk.buf[0];
    f.buf1 = rk.buf[1];
    CUDA_TRY(fast4d_make_maps(f, f.buf0, f.buf1, f.c));
    rk.map_b0 = f.map0;
    rk.map_b1 = f.map1;
    f.st = st;
    f.dt = dt;
    f.loop = 2;
    rk.fi = f;
    rk.fb = f;
    rk.fc = f;
    const PlaneSplit& x = rk.sp;
    if (x.inner) fast4d_bfirst(rk.fi, sms, 0, 0, 0, 0, x.i0, x.i1);
    if (x.bnd) {
      fast4d_bfirst(rk.fb, sms, x.b0, x.e0, x.b1, x.e1, 0, 0);
      fast4d_bfirst(rk.fc, sms, x.b0, x.e0, x.b1, x.e1, x.inner ? x.i0 : 0,
                    x.inner ? x.i1 : 0);
      rk.fc.signal = 1;
      // The persistent sweep fills every SM it runs on (~200 KB of shared
      // memory, 576 threads), so an NCCL kernel launched while it runs could
      // not start before it ends: leave a few SMs to the transfer
      // (HJB_SHARD_COMM_SMS, default 4; dynamic work items rebalance).
      const char* ce = std::getenv("HJB_SHARD_COMM_SMS");
      const int comm_sms = ce ? std::max(0, std::atoi(ce)) : 4;
      const uint32_t cap = static_cast<uint32_t>(std::max(1, sms - comm_sms));
      for (Fast4dArgs* a : {&rk.fi, &rk.fc}) a->blocks = std::min(a->blocks, cap);
    }
    return HJB_OK;
  }
  Ho4dArgs h;
  std::memset(&h, 0, sizeof h);
  h.order = static_cast<int>(geo.R > 3 ? 3 : geo.R);
  h.cbeg = geo.cbeg;
  h.cend = geo.cend;
  fill_lf(p.hm.dm, scheme, galpha, h.lf, h.lp);
  h.tb_fixed = 1;
  ho4d_config(gloc, sms, h);
  if (h.lf && !h.tma)
    return set_err(HJB_ERR_UNSUPPORTED,
                   "solve_sharded: Lax-Friedrichs high order needs the TMA kernels");
  rk.ns = ho_stages(cfg->time_order, rk.stages);
  rk.pe = static_cast<size_t>(ho4d_plane(h));  // stage-buffer plane (ghost layout of h)
  const size_t lbytes = static_cast<size_t>(geo.nloc) * rk.pe * sizeof(double);
  for (int b = 0; b < 4; ++b) {
    CUDA_TRY(bufs[b]->ensure(lbytes));
    CUDA_TRY(cudaMemsetAsync(bufs[b]->p, 0, lbytes, s));
    rk.buf[b] = bufs[b]->d();
  }
  CUDA_TRY(cbuf->ensure(lbytes));
  CUDA_TRY(cudaMemsetAsync(cbuf->p, 0, lbytes, s));
  CUDA_TRY(ho4d_pad(init_slab, rk.buf[0] + geo.cbeg * rk.pe, geo.owned, h, s));
  CUDA_TRY(ho4d_pad(c_slab, cbuf->d() + geo.cbeg * rk.pe, geo.owned, h, s));
  *launches += 2;
  h.tab = p.hm.dm.tab;
  for (int d = 0; d < 4; ++d) {
    h.off_pos[d] = p.hm.dm.row[d].off_pos;
    h.off_neg[d] = p.hm.dm.row[d].off_neg;
    h.off_a[d] = p.hm.dm.row[d].off_a;
    h.off_b[d] = p.hm.dm.row[d].off_b;
  }
  h.c = cbuf->d();
  h.buf0 = rk.buf[0];
  h.buf1 = rk.buf[1];
  h.stage1 = rk.buf[2];
  h.stage2 = rk.buf[3];
  h.st = st;
  h.dt = dt;
  h.loop = 2;
  CUDA_TRY(ho4d_make_maps(h));
  rk.hi = h;
  rk.hb = h;
  rk.hc = h;
  const PlaneSplit& x = rk.sp;
  if (x.inner) ho4d_bfirst(rk.hi, sms, 0, 0, 0, 0, x.i0, x.i1);
  if (x.bnd) {
    ho4d_bfirst(rk.hb, sms, x.b0, x.e0, x.b1, x.e1, 0, 0);
    ho4d_bfirst(rk.hc, sms, x.b0, x.e0, x.b1, x.e1, x.inner ? x.i0 : 0, x.inner ? x.i1 : 0);
    rk.hc.signal = 1;
  }
  return HJB_OK;
}

// the owned planes of the final V -> reference layout
int unpad_rank(const SlabRank& rk, const Prepared& p, long long iters, double* out,
               cudaStream_t s) {
  const double* fin = rk.value(iters) + rk.geo.cbeg * rk.pe;
  if (!rk.ho) {
    const uint64_t rows_owned = static_cast<uint64_t>(rk.geo.owned) * p.g.n[1] * p.g.n[2];
    CUDA_TRY(launch_unpad4(fin, out, rows_owned, p.g.n[3], rk.fi.n3p, s));
  } else {
    CUDA_TRY(ho4d_unpad(fin, out, rk.geo.owned, rk.hi, s));
  }
  return HJB_OK;
}

// -------------------------------------------------------------- transports
int nccl_exchange(Nccl* api, hjb_comm* comm, const SlabRank& rk, double* buf, cudaStream_t s) {
  const Halo h = halo_of(rk.geo);
  const size_t pe = rk.pe, cnt = static_cast<size_t>(h.planes) * pe;
  const int r = comm->rank;
  NCCL_TRY(api->GroupStart());
  if (rk.geo.has_lo) {
    NCCL_TRY(api->Send(buf + h.send_lo * pe, cnt, ncclFloat64_, r - 1, comm->comm, s));
    NCCL_TRY(api->Recv(buf + h.recv_lo * pe, cnt, ncclFloat64_, r - 1, comm->comm, s));
  }
  if (rk.geo.has_hi) {
    NCCL_TRY(api->Send(buf + h.send_hi * pe, cnt, ncclFloat64_, r + 1, comm->comm, s));
    NCCL_TRY(api->Recv(buf + h.recv_hi * pe, cnt, ncclFloat64_, r + 1, comm->comm, s));
  }
  NCCL_TRY(api->GroupEnd());
  return HJB_OK;
}

// In-process ranks on one device: rank r's halo planes receive the planes
// its neighbours send (the same Halo offsets as the NCCL transport).
// bufs[r] = the stage buffer of rank r.
int local_exchange(const std::vector<SlabRank>& rks, const std::vector<double*>& bufs,
                   cudaStream_t s) {
  const int P = static_cast<int>(rks.size());
  for (int r = 0; r < P; ++r) {
    const Halo h = halo_of(rks[r].geo);
    const size_t pe = rks[r].pe;
    const size_t bytes = static_cast<size_t>(h.planes) * pe * sizeof(double);
    if (rks[r].geo.has_lo) {
      const Halo n = halo_of(rks[r - 1].geo);
      CUDA_TRY(cudaMemcpyAsync(bufs[r] + h.recv_lo * pe, bufs[r - 1] + n.send_hi * pe, bytes,
                               cudaMemcpyDeviceToDevice, s));
    }
    if (rks[r].geo.has_hi) {
      const Halo n = halo_of(rks[r + 1].geo);
      CUDA_TRY(cudaMemcpyAsync(bufs[r] + h.recv_hi * pe, bufs[r + 1] + n.send_lo * pe, bytes,
                               cudaMemcpyDeviceToDevice, s));
    }
  }
  return HJB_OK;
}

constexpr int kMaxLocalRanks = 16;
struct RankStates {
  LoopState* st[kMaxLocalRanks];
  int n;
};
// max over the in-process ranks' max|dV| bits, written back to every rank
// (the all-reduce of the NCCL transport)
// slot < 0: maxdv_bits, else maxdv_slot[slot] (pipelined loop)
__global__ void k_reduce_ranks(RankStates p, int slot) {
  if (threadIdx.x != 0) return;
  unsigned long long m = 0ull;
  for (int r = 0; r < p.n; ++r) {
    unsigned long long* a = slot < 0 ? &p.st[r]->maxdv_bits : &p.st[r]->maxdv_slot[slot];
    const unsigned long long b = *(volatile unsigned long long*)a;
    m = b > m ? b : m;
  }
  for (int r = 0; r < p.n; ++r) {
    unsigned long long* a = slot < 0 ? &p.st[r]->maxdv_bits : &p.st[r]->maxdv_slot[slot];
    *a = m;
  }
  __threadfence();
}

// ---- device-side residual all-reduce of the peer-store transport ----
// Every rank owns a mailbox; after a position's sweeps each rank atomically
// max-es its max|dV| bits into slot e % kMboxSlots of EVERY rank's mailbox
// (system-scope atomics over NVLink, or same-device pointers in-process),
// fences, and bumps each mailbox's count.  A rank's stream then waits until
// its own count reaches P * (e / kMboxSlots + 1) (counts are monotonic, never
// reset), takes the max into the loop state's slot, zeroes the mailbox slot
// and runs the epilogue.  A contribution for position m implies (through
// the halo epochs and the epilogue wait of the pipelined loop) that every
// rank has consumed position m - 4, so 8 slots cannot be overwritten early.
constexpr int kMboxSlots = 8;
struct P2PMbox {
  unsigned long long bits[kMboxSlots];
  unsigned int count[kMboxSlots];
};
struct MboxSet {
  P2PMbox* m[kMaxLocalRanks];
  int n;
};
// the CFL scan all-reduce of a peer-store-only communicator: 1 + nd
// non-negative doubles, max-ed as bit patterns (monotonic for values >= +0)
struct ScanMbox {
  unsigned long long bits[kMboxSlots][1 + kMaxDims];
  unsigned int count[kMboxSlots];
};
__global__ void k_scan_contribute(const unsigned long long* mine, MboxSet peers, unsigned int e) {
  if (threadIdx.x != 0) return;
  const int k = static_cast<int>(e % kMboxSlots);
  for (int q = 0; q < peers.n; ++q) {
    ScanMbox* m = reinterpret_cast<ScanMbox*>(peers.m[q]);
    for (int i = 0; i < 1 + kMaxDims; ++i) atomicMax_system(&m->bits[k][i], mine[i]);
  }
  __threadfence_system();
  for (int q = 0; q < peers.n; ++q)
    atomicAdd_system(&reinterpret_cast<ScanMbox*>(peers.m[q])->count[k], 1u);
}
__global__ void k_scan_take(ScanMbox* own, unsigned long long* out, unsigned int e) {
  if (threadIdx.x != 0) return;
  const int k = static_cast<int>(e % kMboxSlots);
  for (int i = 0; i < 1 + kMaxDims; ++i) out[i] = atomicExch_system(&own->bits[k][i], 0ull);
}
// a halo epoch published from the stream (after the V_0 peer copies)
__global__ void k_publish(unsigned int* f0, unsigned int* f1, unsigned int epoch) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  if (f0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f0), "r"(epoch) : "memory");
  if (f1) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f1), "r"(epoch) : "memory");
}

// slot < 0: the source is maxdv_bits, else maxdv_slot[slot]
__global__ void k_p2p_contribute(const LoopState* st, int slot, MboxSet peers, unsigned int e) {
  if (threadIdx.x != 0) return;
  const unsigned long long b =
      slot < 0 ? *(volatile const unsigned long long*)&st->maxdv_bits
               : *(volatile const unsigned long long*)&st->maxdv_slot[slot];
  const int k = static_cast<int>(e % kMboxSlots);
  for (int q = 0; q < peers.n; ++q) atomicMax_system(&peers.m[q]->bits[k], b);
  __threadfence_system();
  for (int q = 0; q < peers.n; ++q) atomicAdd_system(&peers.m[q]->count[k], 1u);
}
__global__ void k_p2p_take(P2PMbox* own, LoopState* st, int slot, unsigned int e) {
  if (threadIdx.x != 0) return;
  const int k = static_cast<int>(e % kMboxSlots);
  const unsigned long long b = atomicExch_system(&own->bits[k], 0ull);
  if (slot < 0)
    st->maxdv_bits = b;
  else
    st->maxdv_slot[slot] = b;
  __threadfence();
}
// HJB_SHARD_OVERLAP=0: the halo transfer runs on the main stream after the
// whole slab is swept (the serial protocol; A/B of the overlap)
bool shard_overlap() {
  const char* e = std::getenv("HJB_SHARD_OVERLAP");
  return !(e && std::strcmp(e, "0") == 0);
}

// HJB_SHARD_PIPE=0: the residual all-reduce + epilogue of sweep k run on the
// main stream before sweep k + 1 (no pipelining)
bool shard_pipeline() {
  const char* e = std::getenv("HJB_SHARD_PIPE");
  return !(e && std::strcmp(e, "0") == 0);
}

// Stream memory operations (driver API, fetched through the runtime like the
// tensor-map encoder): the transfer stream waits until a launch raises
// st->bnd_flag, then re-arms it.  HJB_SHARD_SIGNAL=0 falls back to the
// boundary launch + interior launch split.
typedef CUresult (*PfnValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
  PfnValue32 wait = nullptr, write = nullptr;
};
const MemOps* memops() {
  static MemOps m;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      m.wait = reinterpret_cast<PfnValue32>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      m.write = reinterpret_cast<PfnValue32>(fn);
  });
  return (m.wait && m.write) ? &m : nullptr;
}
bool shard_signal() {
  const char* e = std::getenv("HJB_SHARD_SIGNAL");
  return !(e && std::strcmp(e, "0") == 0) && memops() != nullptr;
}
// peer-store halos (opt-in): HJB_SHARD_P2P=1, first order, stream memory ops
bool shard_p2p() {
  const char* e = std::getenv("HJB_SHARD_P2P");
  return e && std::strcmp(e, "1") == 0 && memops() != nullptr;
}
// the work stream waits until a neighbour has published `epoch` into our flag
int wait_epoch(unsigned int* flag, unsigned int epoch, cudaStream_t s) {
  const CUresult r = memops()->wait(reinterpret_cast<CUstream>(s),
                                    reinterpret_cast<CUdeviceptr>(flag), epoch,
                                    CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? HJB_OK : set_err(HJB_ERR_CUDA, "cuStreamWaitValue32 failed");
}
// contribute, wait for all P contributions, take: the all-reduce of one
// position on stream s; the caller then runs the epilogue
int p2p_allreduce(const LoopState* st, LoopState* st_w, int slot, const MboxSet& peers,
                  P2PMbox* own, int P, unsigned int e, cudaStream_t s) {
  k_p2p_contribute<<<1, 32, 0, s>>>(st, slot, peers, e);
  CUDA_TRY(cudaGetLastError());
  const unsigned int need = static_cast<unsigned int>(P) * (e / kMboxSlots + 1u);
  const CUresult r = memops()->wait(reinterpret_cast<CUstream>(s),
                                    reinterpret_cast<CUdeviceptr>(&own->count[e % kMboxSlots]),
                                    need, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return set_err(HJB_ERR_CUDA, "cuStreamWaitValue32 failed");
  k_p2p_take<<<1, 32, 0, s>>>(own, st_w, slot, e);
  CUDA_TRY(cudaGetLastError());
  return HJB_OK;
}

// Peer-store links between processes: each rank sends its neighbours the
// CUDA IPC handles of its two V buffers and its flag word pair plus the
// plane numbers where it receives halos, over the NCCL communicator; the
// neighbours' allocations are mapped with peer access (NVLink).  The opened
// mappings are closed when the solve returns (IpcPeers).
struct IpcBlob {
  cudaIpcMemHandle_t buf[4];  // V parity 0 / 1, stage1, stage2 (ENO / TVD-RK)
  uint32_t nbuf, recv_lo, recv_hi, pad;
};
static_assert(sizeof(P2PMbox) <= kScanOffset - kMboxOffset, "control block: residual mailbox");
static_assert(sizeof(ScanMbox) <= kBlobOffset - kScanOffset, "control block: scan mailbox");
static_assert(kBlobOffset + sizeof(IpcBlob) <= kCtlBytes, "control block: handle blob");
struct IpcPeers {
  std::vector<void*> opened;
  ~IpcPeers() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
  }
};
// every rank's control block over CUDA IPC, once per communicator: the
// handles are all-gathered as a byte-wise sum (each rank writes only its own
// row of a zeroed P x 64-byte array)
int comm_open_peers(Nccl* api, hjb_comm* comm, cudaStream_t s) {
  if (comm->peers_open) return HJB_OK;
  const int P = comm->nranks;
  if (P > kMaxLocalRanks) return set_err(HJB_ERR_UNSUPPORTED, "peer-store transport: <= 16 ranks");
  std::vector<cudaIpcMemHandle_t> hs(P);
  std::memset(hs.data(), 0, P * sizeof(cudaIpcMemHandle_t));
  CUDA_TRY(cudaIpcGetMemHandle(&hs[comm->rank], comm->p2p_flags));
  DevBuf d;
  CUDA_TRY(d.ensure(P * sizeof(cudaIpcMemHandle_t)));
  CUDA_TRY(cudaMemcpyAsync(d.p, hs.data(), P * sizeof(cudaIpcMemHandle_t), cudaMemcpyHostToDevice, s));
  NCCL_TRY(api->AllReduce(d.p, d.p, P * sizeof(cudaIpcMemHandle_t), 1 /* ncclUint8 */, 0 /* sum */,
                          comm->comm, s));
  CUDA_TRY(cudaMemcpyAsync(hs.data(), d.p, P * sizeof(cudaIpcMemHandle_t), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  comm->peer_ctl.assign(P, nullptr);
  for (int q = 0; q < P; ++q) {
    if (q == comm->rank) {
      comm->peer_ctl[q] = comm->p2p_flags;
      continue;
    }
    CUDA_TRY(cudaIpcOpenMemHandle(&comm->peer_ctl[q], hs[q], cudaIpcMemLazyEnablePeerAccess));
  }
  comm->peers_open = true;
  return HJB_OK;
}
P2PMbox* ctl_mbox(void* ctl) {
  return reinterpret_cast<P2PMbox*>(static_cast<char*>(ctl) + kMboxOffset);
}

int link_ipc_p2p(Nccl* api, hjb_comm* comm, SlabRank& rk, cudaStream_t s, IpcPeers& peers) {
  int rc;
  if ((rc = comm_open_peers(api, comm, s))) return rc;
  IpcBlob mine;
  std::memset(&mine, 0, sizeof mine);
  mine.nbuf = rk.ho ? 4u : 2u;
  for (uint32_t b = 0; b < mine.nbuf; ++b) CUDA_TRY(cudaIpcGetMemHandle(&mine.buf[b], rk.buf[b]));
  const Halo h = halo_of(rk.geo);
  mine.recv_lo = h.recv_lo;
  mine.recv_hi = h.recv_hi;
  DevBuf stage;
  CUDA_TRY(stage.ensure(3 * sizeof(IpcBlob)));  // mine, from below, from above
  IpcBlob* d = static_cast<IpcBlob*>(stage.p);
  CUDA_TRY(cudaMemcpyAsync(d, &mine, sizeof mine, cudaMemcpyHostToDevice, s));
  const int r = comm->rank;
  const size_t nb = sizeof(IpcBlob);
  NCCL_TRY(api->GroupStart());
  if (rk.geo.has_lo) {
    NCCL_TRY(api->Send(d, nb, 0 /* ncclInt8 */, r - 1, comm->comm, s));
    NCCL_TRY(api->Recv(d + 1, nb, 0, r - 1, comm->comm, s));
  }
  if (rk.geo.has_hi) {
    NCCL_TRY(api->Send(d, nb, 0, r + 1, comm->comm, s));
    NCCL_TRY(api->Recv(d + 2, nb, 0, r + 1, comm->comm, s));
  }
  NCCL_TRY(api->GroupEnd());
  IpcBlob nbr[2];
  CUDA_TRY(cudaMemcpyAsync(nbr, d + 1, 2 * nb, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  auto& l = rk.p2p;
  l = SlabRank::P2PLink();
  l.on = true;
  for (int sd = 0; sd < 2; ++sd) {
    if (!(sd == 0 ? rk.geo.has_lo : rk.geo.has_hi)) continue;
    for (uint32_t b = 0; b < nbr[sd].nbuf; ++b) {
      void* p = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&p, nbr[sd].buf[b], cudaIpcMemLazyEnablePeerAccess));
      peers.opened.push_back(p);
      l.peer_buf[sd][b] = static_cast<double*>(p);
    }
    void* f = comm->peer_ctl[sd == 0 ? comm->rank - 1 : comm->rank + 1];
    // our first send plane lands on the lower neighbour's first upper-halo
    // plane, the upper neighbour's on its first lower-halo plane
    l.dst0[sd] = sd == 0 ? nbr[sd].recv_hi : nbr[sd].recv_lo;
    l.peer_flag[sd] = static_cast<unsigned int*>(f) + (sd == 0 ? 1 : 0);
    l.own_flag[sd] = comm->p2p_flags + sd;
  }
  return HJB_OK;
}

// Per-solve buffer handles of a peer-store-only communicator: each rank
// writes its blob into its own control block and bumps its blob epoch; the
// neighbours poll that epoch through their mapping and then read the blob
// (host-side, bounded wait: an absent neighbour is an error, not a hang).
int link_blob_p2p(hjb_comm* comm, SlabRank& rk, IpcPeers& peers) {
  IpcBlob mine;
  std::memset(&mine, 0, sizeof mine);
  mine.nbuf = rk.ho ? 4u : 2u;
  for (uint32_t b = 0; b < mine.nbuf; ++b) CUDA_TRY(cudaIpcGetMemHandle(&mine.buf[b], rk.buf[b]));
  const Halo h = halo_of(rk.geo);
  mine.recv_lo = h.recv_lo;
  mine.recv_hi = h.recv_hi;
  char* own = reinterpret_cast<char*>(comm->p2p_flags);
  CUDA_TRY(cudaMemcpy(own + kBlobOffset, &mine, sizeof mine, cudaMemcpyHostToDevice));
  const unsigned int ep = ++comm->blob_seq;
  CUDA_TRY(cudaMemcpy(own + kBlobFlagOffset, &ep, sizeof ep, cudaMemcpyHostToDevice));
  auto& l = rk.p2p;
  l = SlabRank::P2PLink();
  l.on = true;
  for (int sd = 0; sd < 2; ++sd) {
    if (!(sd == 0 ? rk.geo.has_lo : rk.geo.has_hi)) continue;
    const int q = sd == 0 ? comm->rank - 1 : comm->rank + 1;
    char* pc = static_cast<char*>(comm->peer_ctl[q]);
    unsigned int seen = 0;
    for (int it = 0; it < 1200000; ++it) {  // ~2 min at 100 us per poll
      CUDA_TRY(cudaMemcpy(&seen, pc + kBlobFlagOffset, sizeof seen, cudaMemcpyDeviceToHost));
      if (seen >= ep) break;
      std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
    if (seen < ep) return set_err(HJB_ERR_RUNTIME, "peer-store link: neighbour did not publish");
    IpcBlob nb;
    CUDA_TRY(cudaMemcpy(&nb, pc + kBlobOffset, sizeof nb, cudaMemcpyDeviceToHost));
    for (uint32_t b = 0; b < nb.nbuf; ++b) {
      void* p = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&p, nb.buf[b], cudaIpcMemLazyEnablePeerAccess));
      peers.opened.push_back(p);
      l.peer_buf[sd][b] = static_cast<double*>(p);
    }
    l.dst0[sd] = sd == 0 ? nb.recv_hi : nb.recv_lo;
    l.peer_flag[sd] = reinterpret_cast<unsigned int*>(pc) + (sd == 0 ? 1 : 0);
    l.own_flag[sd] = comm->p2p_flags + sd;
  }
  return HJB_OK;
}

// the peer-store links of in-process ranks (same device: the neighbours'
// buffers and flags are plain device pointers)
void link_local_p2p(std::vector<SlabRank>& rks, unsigned int* flags) {
  const int P = static_cast<int>(rks.size());
  for (int r = 0; r < P; ++r) {
    auto& l = rks[r].p2p;
    l = SlabRank::P2PLink();
    l.on = true;
    if (r > 0) {
      for (int b = 0; b < 4; ++b) l.peer_buf[0][b] = rks[r - 1].buf[b];
      l.dst0[0] = halo_of(rks[r - 1].geo).recv_hi;
      l.peer_flag[0] = flags + 2 * (r - 1) + 1;  // the lower rank's "from above"
      l.own_flag[0] = flags + 2 * r;
    }
    if (r < P - 1) {
      for (int b = 0; b < 4; ++b) l.peer_buf[1][b] = rks[r + 1].buf[b];
      l.dst0[1] = halo_of(rks[r + 1].geo).recv_lo;
      l.peer_flag[1] = flags + 2 * (r + 1);  // the upper rank's "from below"
      l.own_flag[1] = flags + 2 * r + 1;
    }
  }
}
// the transfer stream waits for / re-arms one rank's boundary flag
int wait_flag(LoopState* st, cudaStream_t s) {
  const CUresult r = memops()->wait(reinterpret_cast<CUstream>(s),
                                    reinterpret_cast<CUdeviceptr>(&st->bnd_flag), 1u,
                                    CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? HJB_OK : set_err(HJB_ERR_CUDA, "cuStreamWaitValue32 failed");
}
int rearm_flag(LoopState* st, cudaStream_t s) {
  CUresult r = memops()->write(reinterpret_cast<CUstream>(s),
                               reinterpret_cast<CUdeviceptr>(&st->bnd_done), 0u,
                               CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r == CUDA_SUCCESS)
    r = memops()->write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(&st->bnd_flag),
                        0u, CU_STREAM_WRITE_VALUE_DEFAULT);
  return r == CUDA_SUCCESS ? HJB_OK : set_err(HJB_ERR_CUDA, "cuStreamWriteValue32 failed");
}

// Streams and events of the sharded loop.  The sweep KERNELS run on a work
// stream W; halo transfers, the residual reduction (NCCL all-reduce or the
// in-process kernel) and the epilogue run on the capture's origin stream S,
// so every NCCL call stays on the stream the caller captures (a 1-rank
// all-reduce issued from a joined side stream hung inside the conditional
// graph on the B200 pool).
//
// Per position k and RK stage q:  W: boundary planes -> S: send/recv of the
// stage output's boundary planes || W: interior planes; the next stage waits
// for the transfer.  After the last stage S reduces max|dV| and runs the
// epilogue.  Pipelined residual (default): position k accumulates into
// st->maxdv_slot[k & 1] and W starts position k + 1 as soon as its halo is
// in, while S still reduces position k.  Position k reads V_k and writes
// V_{k+1} over V_{k-1}; if epilogue k - 2 stopped the loop V_{k-1} is the
// result, so W waits for epilogue k - 2 first.  The one speculative sweep
// after the stopping one overwrites only the previous iterate, and its
// epilogue returns early (done), so iteration count, history and status are
// the unpipelined ones.
struct LoopStreams {
  cudaStream_t work = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_bnd = nullptr, ev_xs = nullptr, ev_int = nullptr;
  cudaEvent_t ev_xl[2] = {nullptr, nullptr}, ev_epi[2] = {nullptr, nullptr};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ~LoopStreams() {
    for (cudaEvent_t e : {ev_fork, ev_bnd, ev_xs, ev_int, ev_xl[0], ev_xl[1], ev_epi[0],
                          ev_epi[1], e0, e1})
      if (e) cudaEventDestroy(e);
    if (work) cudaStreamDestroy(work);
  }
  cudaError_t init() {
    cudaError_t e = cudaStreamCreateWithFlags(&work, cudaStreamNonBlocking);
    for (cudaEvent_t* ev : {&ev_fork, &ev_bnd, &ev_xs, &ev_int, &ev_xl[0], &ev_xl[1], &ev_epi[0],
                            &ev_epi[1]})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    return e;
  }
};

// What one loop position does, per transport (NCCL ranks / in-process ranks)
struct PositionOps {
  int ns = 1;                  // RK stages
  bool bnd = false, inner = true, xfer = false;
  // signal: one launch per stage (boundary items first); the transfer
  // stream waits on the launch's bnd_flag (wait_bnd), moves the halos and
  // re-arms the flag (reset_bnd).  Otherwise a boundary launch, then the
  // transfer (after the launch) || an interior launch.
  bool signal = false;
  std::function<int(cudaStream_t s)> wait_bnd, reset_bnd;
  // peer-store halos: the sweep kernels store the boundary planes into the
  // neighbours' halos and publish an epoch; before each stage the work
  // stream waits for the neighbours' epoch of the stage it reads (p2p_wait)
  // and re-arms the boundary counter (reset_bnd); no transfer on S
  bool p2p = false;
  std::function<int(cudaStream_t s)> p2p_wait;
  // sweep kernels of stage q on stream s (mode kBnd / kInner / kBoth)
  std::function<int(int k, int q, int mode, bool pipe, cudaStream_t s)> sweep;
  // halo transfer of stage q's output, on s
  std::function<int(int k, int q, cudaStream_t s)> exchange;
  // residual reduction + epilogue of position k, on s
  std::function<int(int k, bool pipe, cudaGraphConditionalHandle h, int use, cudaStream_t s)>
      finish;
};

int run_position(LoopStreams& ls, cudaStream_t S, const PositionOps& op, int k, bool overlap,
                 bool pipe, cudaGraphConditionalHandle h, int use) {
  int e;
  if (!overlap) {  // serial: every kernel, then the transfer, on S; no pipelining
    for (int q = 0; q < op.ns; ++q) {
      if (op.bnd && (e = op.sweep(k, q, kBnd, false, S))) return e;
      if (op.inner && (e = op.sweep(k, q, kInner, false, S))) return e;
      if (op.xfer && (e = op.exchange(k, q, S))) return e;
    }
    return op.finish(k, false, h, use, S);
  }
  cudaStream_t W = ls.work;
  if (k == 0) {  // W joins the capture (position 0 follows everything before)
    CUDA_TRY(cudaEventRecord(ls.ev_fork, S));
    CUDA_TRY(cudaStreamWaitEvent(W, ls.ev_fork, 0));
  } else {
    if (op.xfer && !op.p2p) CUDA_TRY(cudaStreamWaitEvent(W, ls.ev_xl[(k - 1) & 1], 0));  // halo of V_k
    if (!pipe) CUDA_TRY(cudaStreamWaitEvent(W, ls.ev_epi[(k - 1) & 1], 0));
    else if (k >= 2) CUDA_TRY(cudaStreamWaitEvent(W, ls.ev_epi[k & 1], 0));
  }
  for (int q = 0; q < op.ns; ++q) {
    if (op.p2p) {  // one launch per stage; its kernels store the halos themselves
      if ((e = op.p2p_wait(W))) return e;
      if ((e = op.reset_bnd(W))) return e;
      if ((e = op.sweep(k, q, kBoth, pipe, W))) return e;
      continue;
    }
    if (op.xfer && op.signal) {  // one launch; the transfer starts on its flag
      if ((e = op.sweep(k, q, kBoth, pipe, W))) return e;
      if ((e = op.wait_bnd(S))) return e;
      if ((e = op.exchange(k, q, S))) return e;
      if ((e = op.reset_bnd(S))) return e;
      CUDA_TRY(cudaEventRecord(q == op.ns - 1 ? ls.ev_xl[k & 1] : ls.ev_xs, S));
      if (q < op.ns - 1) CUDA_TRY(cudaStreamWaitEvent(W, ls.ev_xs, 0));
      continue;
    }
    if (op.bnd && (e = op.sweep(k, q, kBnd, pipe, W))) return e;
    if (op.xfer) {
      CUDA_TRY(cudaEventRecord(ls.ev_bnd, W));
      CUDA_TRY(cudaStreamWaitEvent(S, ls.ev_bnd, 0));
      if ((e = op.exchange(k, q, S))) return e;
      CUDA_TRY(cudaEventRecord(q == op.ns - 1 ? ls.ev_xl[k & 1] : ls.ev_xs, S));
    }
    if (op.inner && (e = op.sweep(k, q, kInner, pipe, W))) return e;
    if (op.xfer && q < op.ns - 1) CUDA_TRY(cudaStreamWaitEvent(W, ls.ev_xs, 0));
  }
  CUDA_TRY(cudaEventRecord(ls.ev_int, W));
  CUDA_TRY(cudaStreamWaitEvent(S, ls.ev_int, 0));  // also joins W back into S
  if ((e = op.finish(k, pipe, h, use, S))) return e;
  CUDA_TRY(cudaEventRecord(ls.ev_epi[k & 1], S));
  return HJB_OK;
}

// result fields from the loop state of the reporting rank
int fill_result(hjb_context* ctx, float ms, hjb_solve_result* res) {
  CUDA_TRY(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(LoopState), cudaMemcpyDeviceToHost,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  const LoopState& st = *ctx->st_host;
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
  return HJB_OK;
}

// validation, slab-thickness check and the CFL scan shared by both drivers;
// `allreduce` (may be null) turns the local scan into the global one
int sharded_prologue(hjb_context* ctx, const hjb_grid* gi, const hjb_model* mi,
                     const hjb_dbounds* db, const hjb_solve_config* cfg, int P, Prepared& p,
                     Scan& s, uint32_t& R, const std::function<int(Scan&)>& allreduce,
                     const DevGrid* scan_grid_override) {
  int rc;
  CUDA_TRY(cudaSetDevice(ctx->device));
  if ((rc = validate_config(cfg))) return rc;
  if (cfg->target)
    return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: no target set (use solve)");
  if ((rc = prepare(ctx, gi, mi, db, p))) return rc;
  if (p.shape < 0)
    return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: model/grid outside the 4D fast path");
  if (fast4d_shape(p.g, p.hm.dm, scheme_of(cfg)) != p.shape)
    return set_err(HJB_ERR_UNSUPPORTED,
                   "solve_sharded: Lax-Friedrichs needs one input term per row of the 4D model");
  const bool high_order = cfg->spatial_order > 1 || cfg->time_order > 1;
  if (high_order && p.shape == kShapeGen)
    return set_err(HJB_ERR_UNSUPPORTED,
                   "solve_sharded: ENO / TVD-RK slabs need one of the compiled 4D model shapes");
  if (p.shape == kShapeGen) {
    Fast4dArgs probe;
    std::memset(&probe, 0, sizeof probe);
    fast4d_gen_rows(p.hm.dm, probe);
    if (probe.gx0)  // slab-local plane numbers would index the x0 tables
      return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: a model row depends on x0 (the slab axis)");
  }
  R = high_order ? static_cast<uint32_t>(cfg->spatial_order < 1 ? 1 : cfg->spatial_order) : 1u;
  // Every rank must reject a too-thin partition BEFORE the first collective:
  // balanced slabs differ by one plane, so a per-rank check would let the
  // thicker ranks enter NCCL while a thin one returns (a hang, not an error).
  // The smallest slab is floor(n0 / P) planes on every rank's view.
  if (P > 1 && static_cast<int64_t>(p.g.n[0]) / P < static_cast<int64_t>(R))
    return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: slab thinner than the ENO halo");
  if ((rc = run_scan(ctx, scan_grid_override ? *scan_grid_override : p.g, p.hm.dm, s))) return rc;
  if (allreduce && (rc = allreduce(s))) return rc;
  if (!(s.max_speed_sum > 0.0))
    return set_err(HJB_ERR_RUNTIME, "solve: flow is identically zero on the grid");
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

int hjb_slab_plan(int64_t n0, int32_t nranks, int32_t rank, int32_t halo, int64_t* o) {
  if (!o || halo < 1) return set_err(HJB_ERR_INVALID_ARGUMENT, "slab_plan: bad arguments");
  int64_t b, e;
  int rc = hjb_slab_partition(n0, nranks, rank, &b, &e);
  if (rc) return rc;
  const SlabGeom g = slab_geom(static_cast<uint32_t>(n0), nranks, rank, static_cast<uint32_t>(halo));
  const Halo h = halo_of(g);
  const PlaneSplit x = plane_split(g);
  const int64_t v[16] = {g.owned, g.nloc, g.cbeg, g.cend, g.gbeg,
                         g.has_lo ? (int64_t)h.send_lo : -1, g.has_lo ? (int64_t)h.recv_lo : -1,
                         g.has_hi ? (int64_t)h.send_hi : -1, g.has_hi ? (int64_t)h.recv_hi : -1,
                         h.planes, x.b0, x.e0, x.b1, x.e1, x.i0, x.i1};
  std::memcpy(o, v, sizeof v);
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
  // the flags must be their own cudaMalloc allocation (IPC handles map whole
  // allocations) and zero before any neighbour can write them: the first
  // peer write happens after the first halo exchange, which every rank
  // enters only after this comm_create returned everywhere
  if (cudaMalloc(&c->p2p_flags, kCtlBytes) != cudaSuccess ||
      cudaMemset(c->p2p_flags, 0, kCtlBytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    if (c->p2p_flags) cudaFree(c->p2p_flags);
    api->CommDestroy(c->comm);
    delete c;
    return set_err(HJB_ERR_CUDA, "comm_create: peer-store flag allocation failed");
  }
  *out = c;
  return HJB_OK;
}

int hjb_p2p_comm_create(hjb_context* ctx, int32_t nranks, int32_t rank, hjb_comm** out) {
  if (!ctx || !out) return set_err(HJB_ERR_INVALID_ARGUMENT, "p2p_comm_create: null");
  if (nranks < 1 || nranks > kMaxLocalRanks || rank < 0 || rank >= nranks)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "p2p_comm_create: 1 <= nranks <= 16, 0 <= rank < nranks");
  CUDA_TRY(cudaSetDevice(ctx->device));
  hjb_comm* c = new hjb_comm();
  c->nranks = nranks;
  c->rank = rank;
  if (cudaMalloc(&c->p2p_flags, kCtlBytes) != cudaSuccess ||
      cudaMemset(c->p2p_flags, 0, kCtlBytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    if (c->p2p_flags) cudaFree(c->p2p_flags);
    delete c;
    return set_err(HJB_ERR_CUDA, "p2p_comm_create: control block allocation failed");
  }
  *out = c;
  return HJB_OK;
}

int hjb_comm_ctl_handle(hjb_comm* c, void* out64) {
  if (!c || !out64) return set_err(HJB_ERR_INVALID_ARGUMENT, "comm_ctl_handle: null");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->p2p_flags));
  std::memcpy(out64, &h, sizeof h);
  return HJB_OK;
}

int hjb_comm_open_peers(hjb_comm* c, const void* handles) {
  if (!c || !handles) return set_err(HJB_ERR_INVALID_ARGUMENT, "comm_open_peers: null");
  if (c->peers_open) return HJB_OK;
  const cudaIpcMemHandle_t* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  c->peer_ctl.assign(c->nranks, nullptr);
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      c->peer_ctl[q] = c->p2p_flags;
      continue;
    }
    CUDA_TRY(cudaIpcOpenMemHandle(&c->peer_ctl[q], hs[q], cudaIpcMemLazyEnablePeerAccess));
  }
  c->peers_open = true;
  return HJB_OK;
}

int hjb_comm_destroy(hjb_comm* c) {
  if (!c) return HJB_OK;
  for (int q = 0; q < static_cast<int>(c->peer_ctl.size()); ++q)
    if (q != c->rank && c->peer_ctl[q]) cudaIpcCloseMemHandle(c->peer_ctl[q]);
  if (c->comm && nccl() && nccl()->CommDestroy) nccl()->CommDestroy(c->comm);
  if (c->p2p_flags) cudaFree(c->p2p_flags);
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
  if (p.shape < 0 || p.shape == kShapeGen)
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
  // peer-store-only communicator: no NCCL anywhere (first order)
  const bool p2p_only = comm->comm == nullptr;
  Nccl* api = p2p_only ? nullptr : nccl();
  if (!p2p_only && !api) return set_err(HJB_ERR_NCCL, "libnccl.so.2 not loadable");
  if (p2p_only && comm->nranks == 1 && !comm->peers_open) {  // a single rank is its own peer
    comm->peer_ctl.assign(1, comm->p2p_flags);
    comm->peers_open = true;
  }
  if (p2p_only && (!comm->peers_open || !memops()))
    return set_err(HJB_ERR_INVALID_ARGUMENT, "solve_sharded: open the peers first (hjb_comm_open_peers)");
  const int P = comm->nranks, r = comm->rank;
  Prepared p;
  Scan s;
  uint32_t R = 1;
  // CFL scan over the slab + all-reduce(max): rows of the fast path never
  // depend on x0, so the slab's local grid gives the global values
  DevGrid gl;
  auto allreduce = [&](Scan& sc) -> int {
    unsigned long long bits[1 + kMaxDims];
    std::memcpy(bits, &sc.max_speed_sum, sizeof(double));
    std::memcpy(bits + 1, sc.max_alpha, kMaxDims * sizeof(double));
    unsigned long long* dbits = reinterpret_cast<unsigned long long*>(ctx->scratch.d());
    CUDA_TRY(cudaMemcpyAsync(dbits, bits, sizeof bits, cudaMemcpyHostToDevice, ctx->stream));
    if (p2p_only) {  // through every rank's scan mailbox
      MboxSet ms;
      ms.n = P;
      for (int q = 0; q < P; ++q)
        ms.m[q] = reinterpret_cast<P2PMbox*>(static_cast<char*>(comm->peer_ctl[q]) + kScanOffset);
      const unsigned int e = comm->scan_seq++;
      k_scan_contribute<<<1, 32, 0, ctx->stream>>>(dbits, ms, e);
      CUDA_TRY(cudaGetLastError());
      ScanMbox* own = reinterpret_cast<ScanMbox*>(reinterpret_cast<char*>(comm->p2p_flags) + kScanOffset);
      int we = wait_epoch(&own->count[e % kMboxSlots],
                          static_cast<unsigned int>(P) * (e / kMboxSlots + 1u), ctx->stream);
      if (we) return we;
      k_scan_take<<<1, 32, 0, ctx->stream>>>(own, dbits, e);
      CUDA_TRY(cudaGetLastError());
    } else {
      NCCL_TRY(api->AllReduce(dbits, dbits, 1 + kMaxDims, ncclUint64_, ncclMax_, comm->comm,
                              ctx->stream));
    }
    CUDA_TRY(cudaMemcpyAsync(bits, dbits, sizeof bits, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    std::memcpy(&sc.max_speed_sum, bits, sizeof(double));
    std::memcpy(sc.max_alpha, bits + 1, kMaxDims * sizeof(double));
    return HJB_OK;
  };
  {
    // the slab's own grid for the scan (needs p.g: validate/prepare first)
    CUDA_TRY(cudaSetDevice(ctx->device));
    if ((rc = validate_config(cfg))) return rc;
    DevGrid g;
    if ((rc = make_grid(gi, g))) return rc;
    if (g.nd != 4)
      return set_err(HJB_ERR_UNSUPPORTED, "solve_sharded: model/grid outside the 4D fast path");
    int64_t b, e;
    if ((rc = hjb_slab_partition(g.n[0], P, r, &b, &e))) return rc;
    gl = g;
    gl.n[0] = static_cast<uint32_t>(e - b);
    gl.size = gl.n[0] * gl.stride[0];
    gl.divs[0].init(gl.n[0]);
  }
  if ((rc = sharded_prologue(ctx, gi, mi, db, cfg, P, p, s, R, allreduce, &gl))) return rc;
  const double dt = cfg->cfl_factor / s.max_speed_sum;
  hjb_solve_result local;
  std::memset(&local, 0, sizeof local);
  if (!res) res = &local;
  res->dt = dt;
  res->nodes_per_sweep = p.g.size;
  res->iterations = 0;
  res->converged = 0;
  const SlabGeom geo = slab_geom(p.g.n[0], P, r, R);
  if (cfg->max_iters == 0) {
    CUDA_TRY(cudaMemcpyAsync(value_slab_out, init_slab,
                             static_cast<size_t>(geo.owned) * p.g.stride[0] * sizeof(double),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return HJB_OK;
  }
  SlabRank rk;
  DevBuf* const bufs[4] = {&ctx->v0, &ctx->v1, &ctx->v2, &ctx->v3};
  if ((rc = setup_rank(ctx->device, p, cfg, dt, s.max_alpha, geo, bufs, &ctx->pcbuf, ctx->st,
                       init_slab, c_slab, ctx->stream, rk, &ctx->launches)))
    return rc;
  const long long cap =
      std::min<long long>(cfg->max_iters, std::max<long long>(res->history_capacity, 1));
  CUDA_TRY(ctx->hist.ensure(cap * sizeof(double)));
  CUDA_TRY(ctx->whist.ensure(cap * sizeof(double)));
  CUDA_TRY(launch_loop_init(ctx->st, cfg->max_iters, dt, cfg->tolerance,
                            cfg->time_horizon > 0.0 ? cfg->time_horizon : 0.0, cap,
                            ctx->hist.d(), ctx->whist.d(), ctx->stream));
  ++ctx->launches;
  LoopStreams ls;
  CUDA_TRY(ls.init());
  // halos of V_0 (afterwards every stage output travels right after its
  // boundary planes are swept)
  IpcPeers ipc;
  if (P > 1 && p2p_only) {
    // buffer handles through the control blocks, then V_0's boundary planes
    // copied into the neighbours' halos and published as one epoch
    if ((rc = link_blob_p2p(comm, rk, ipc))) return rc;
    const Halo h = halo_of(rk.geo);
    const size_t bytes = static_cast<size_t>(h.planes) * rk.pe * sizeof(double);
    if (rk.geo.has_lo)
      CUDA_TRY(cudaMemcpyAsync(rk.p2p.peer_buf[0][0] + rk.p2p.dst0[0] * rk.pe,
                               rk.buf[0] + h.send_lo * rk.pe, bytes, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    if (rk.geo.has_hi)
      CUDA_TRY(cudaMemcpyAsync(rk.p2p.peer_buf[1][0] + rk.p2p.dst0[1] * rk.pe,
                               rk.buf[0] + h.send_hi * rk.pe, bytes, cudaMemcpyDeviceToDevice,
                               ctx->stream));
    k_publish<<<1, 32, 0, ctx->stream>>>(rk.p2p.peer_flag[0], rk.p2p.peer_flag[1],
                                         ++comm->p2p_seq);
    CUDA_TRY(cudaGetLastError());
  } else if (P > 1 && (rc = nccl_exchange(api, comm, rk, rk.buf[0], ctx->stream))) {
    return rc;
  }
  unsigned long long* maxbits = &ctx->st->maxdv_bits;
  const bool overlap = shard_overlap();
  const bool pipe = shard_pipeline();
  const int body = rk.ho ? 2 : 8;  // even: buffer parity of position k == iteration parity
  long long per_pos = 0;
  PositionOps op;
  op.ns = rk.ns;
  op.bnd = rk.sp.bnd;
  op.inner = rk.sp.inner;
  op.xfer = P > 1;
  op.signal = op.xfer && shard_signal();
  op.wait_bnd = [&](cudaStream_t s) -> int { return wait_flag(ctx->st, s); };
  op.reset_bnd = [&](cudaStream_t s) -> int { return rearm_flag(ctx->st, s); };
  // peer-store halos (opt-in with NCCL, always without it; first order): the
  // neighbours' buffers and flags mapped over CUDA IPC; the kernels store
  // the halo planes over NVLink
  if (P > 1 && p2p_only) {
    op.p2p = true;
  } else if (P > 1 && shard_p2p()) {
    if ((rc = link_ipc_p2p(api, comm, rk, ctx->stream, ipc))) return rc;
    op.p2p = true;
  }
  op.p2p_wait = [&](cudaStream_t s) -> int {
    if (comm->p2p_seq == 0) return HJB_OK;  // nothing published yet (V_0 came by NCCL)
    for (int sd = 0; sd < 2; ++sd)
      if (rk.p2p.own_flag[sd]) {
        int e = wait_epoch(rk.p2p.own_flag[sd], comm->p2p_seq, s);
        if (e) return e;
      }
    return HJB_OK;
  };
  op.sweep = [&](int k, int q, int mode, bool pp, cudaStream_t s) -> int {
    if (op.p2p) rk.p2p.epoch = comm->p2p_seq + 1;
    CUDA_TRY(rk.launch(k, q, mode, pp ? &ctx->st->maxdv_slot[k & 1] : maxbits, s));
    if (op.p2p) ++comm->p2p_seq;
    ++per_pos;
    return HJB_OK;
  };
  op.exchange = [&](int k, int q, cudaStream_t s) -> int {
    return nccl_exchange(api, comm, rk, rk.stage_out(k, q), s);
  };
  op.finish = [&](int k, bool pp, cudaGraphConditionalHandle hd, int use, cudaStream_t s) -> int {
    unsigned long long* slot = pp ? &ctx->st->maxdv_slot[k & 1] : maxbits;
    if (op.p2p || p2p_only) {  // device-side all-reduce over the ranks' mailboxes (NVLink atomics)
      MboxSet ms;
      ms.n = P;
      for (int q = 0; q < P; ++q) ms.m[q] = ctl_mbox(comm->peer_ctl[q]);
      int e = p2p_allreduce(ctx->st, ctx->st, pp ? (k & 1) : -1, ms, ctl_mbox(comm->p2p_flags), P,
                            comm->res_seq++, s);
      if (e) return e;
      CUDA_TRY(launch_epilogue(ctx->st, hd, use, s, pp ? slot : nullptr));
      per_pos += 3;
      return HJB_OK;
    }
    NCCL_TRY(api->AllReduce(slot, slot, 1, ncclUint64_, ncclMax_, comm->comm, s));
    CUDA_TRY(launch_epilogue(ctx->st, hd, use, s, pp ? slot : nullptr));
    ++per_pos;
    return HJB_OK;
  };
  auto step = [&](int k, cudaGraphConditionalHandle hd, int use) -> int {
    per_pos = 0;
    return run_position(ls, ctx->stream, op, k, overlap, pipe, hd, use);
  };
  CUDA_TRY(cudaEventRecord(ls.e0, ctx->stream));
  if ((rc = run_eager_loop(ctx, body, step))) return rc;
  CUDA_TRY(cudaEventRecord(ls.e1, ctx->stream));
  CUDA_TRY(cudaEventSynchronize(ls.e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ls.e0, ls.e1);
  if ((rc = fill_result(ctx, ms, res))) return rc;
  res->kernel = rk.ho ? HJB_KERNEL_HO4D : HJB_KERNEL_FAST4D;
  ctx->launches += per_pos * (res->iterations + 2 * body);
  const LoopState& st = *ctx->st_host;
  if ((rc = unpad_rank(rk, p, st.iter, value_slab_out, ctx->stream))) return rc;
  ++ctx->launches;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (st.status == HJB_ERR_DIVERGED)
    return set_err(HJB_ERR_DIVERGED, "solve: diverging (residual grew 10x above its minimum)");
  return HJB_OK;
}

int hjb_solve_sharded_local_dev(hjb_context* ctx, int32_t nranks, const hjb_grid* gi,
                                const hjb_model* mi, const hjb_dbounds* db, const double* init,
                                const double* c, const hjb_solve_config* cfg, double* value_out,
                                hjb_solve_result* res) {
  int rc;
  if (!ctx) return set_err(HJB_ERR_INVALID_ARGUMENT, "context: null");
  if (nranks < 1 || nranks > kMaxLocalRanks)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "solve_sharded_local: 1..16 ranks");
  const int P = nranks;
  Prepared p;
  Scan s;
  uint32_t R = 1;
  if ((rc = sharded_prologue(ctx, gi, mi, db, cfg, P, p, s, R, nullptr, nullptr))) return rc;
  if (static_cast<int64_t>(p.g.n[0]) < P)
    return set_err(HJB_ERR_INVALID_ARGUMENT, "slab_partition: need 0 <= rank < nranks <= n0");
  const double dt = cfg->cfl_factor / s.max_speed_sum;
  hjb_solve_result local;
  std::memset(&local, 0, sizeof local);
  if (!res) res = &local;
  res->dt = dt;
  res->nodes_per_sweep = p.g.size;
  res->iterations = 0;
  res->converged = 0;
  if (cfg->max_iters == 0) {
    CUDA_TRY(cudaMemcpyAsync(value_out, init, static_cast<size_t>(p.g.size) * sizeof(double),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return HJB_OK;
  }
  const size_t s0 = p.g.stride[0];
  // per-rank buffers (rank 0 uses the context's, so its loop state drives
  // the loop and the result), loop states of ranks 1..P-1
  std::vector<std::unique_ptr<DevBuf>> own;
  DevBuf states;
  CUDA_TRY(states.ensure(static_cast<size_t>(P) * sizeof(LoopState)));
  std::vector<SlabRank> rks(P);
  RankStates rs;
  rs.n = P;
  for (int r = 0; r < P; ++r) {
    const SlabGeom geo = slab_geom(p.g.n[0], P, r, R);
    DevBuf* bufs[4];
    DevBuf* cb;
    if (r == 0) {
      bufs[0] = &ctx->v0;
      bufs[1] = &ctx->v1;
      bufs[2] = &ctx->v2;
      bufs[3] = &ctx->v3;
      cb = &ctx->pcbuf;
    } else {
      for (int b = 0; b < 4; ++b) {
        own.emplace_back(new DevBuf());
        bufs[b] = own.back().get();
      }
      own.emplace_back(new DevBuf());
      cb = own.back().get();
    }
    LoopState* st = r == 0 ? ctx->st : reinterpret_cast<LoopState*>(states.p) + r;
    rs.st[r] = st;
    if ((rc = setup_rank(ctx->device, p, cfg, dt, s.max_alpha, geo, bufs, cb, st,
                         init + geo.gbeg * s0, c + geo.gbeg * s0, ctx->stream, rks[r],
                         &ctx->launches)))
      return rc;
    if (rks[r].pe != rks[0].pe)
      return set_err(HJB_ERR_RUNTIME, "solve_sharded_local: plane layouts differ across ranks");
  }
  const long long cap =
      std::min<long long>(cfg->max_iters, std::max<long long>(res->history_capacity, 1));
  CUDA_TRY(ctx->hist.ensure(cap * sizeof(double)));
  CUDA_TRY(ctx->whist.ensure(cap * sizeof(double)));
  for (int r = 0; r < P; ++r) {
    CUDA_TRY(launch_loop_init(rs.st[r], cfg->max_iters, dt, cfg->tolerance,
                              cfg->time_horizon > 0.0 ? cfg->time_horizon : 0.0,
                              r == 0 ? cap : 0, r == 0 ? ctx->hist.d() : nullptr,
                              r == 0 ? ctx->whist.d() : nullptr, ctx->stream));
    ++ctx->launches;
  }
  LoopStreams ls;
  CUDA_TRY(ls.init());
  std::vector<double*> xb(P);
  for (int r = 0; r < P; ++r) xb[r] = rks[r].buf[0];
  if (P > 1 && (rc = local_exchange(rks, xb, ctx->stream))) return rc;
  long long per_pos = 0;
  const bool overlap = shard_overlap();
  const bool pipe = shard_pipeline();
  const int body = rks[0].ho ? 2 : 8;
  bool any_bnd = false, any_inner = false;
  for (int r = 0; r < P; ++r) {
    any_bnd = any_bnd || rks[r].sp.bnd;
    any_inner = any_inner || rks[r].sp.inner;
  }
  PositionOps op;
  op.ns = rks[0].ns;
  op.bnd = any_bnd;
  op.inner = any_inner;
  op.xfer = P > 1;
  // in-process ranks share one host thread: the signalling protocol's eager
  // loop would be host-bound there, so it is opt-in (HJB_SHARD_SIGNAL=1)
  {
    const char* e = std::getenv("HJB_SHARD_SIGNAL");
    op.signal = op.xfer && e && std::strcmp(e, "1") == 0 && shard_signal();
  }
  op.wait_bnd = [&](cudaStream_t s) -> int {
    for (int r = 0; r < P; ++r) {
      int e = wait_flag(rs.st[r], s);
      if (e) return e;
    }
    return HJB_OK;
  };
  op.reset_bnd = [&](cudaStream_t s) -> int {
    for (int r = 0; r < P; ++r) {
      int e = rearm_flag(rs.st[r], s);
      if (e) return e;
    }
    return HJB_OK;
  };
  // peer-store halos (opt-in, first order): the kernels write the
  // neighbours' halo planes; one epoch counter for all ranks
  DevBuf p2p_flags;
  unsigned int p2p_seq = 0;
  if (P > 1 && shard_p2p()) {
    CUDA_TRY(p2p_flags.ensure(2 * static_cast<size_t>(P) * sizeof(unsigned int)));
    CUDA_TRY(cudaMemsetAsync(p2p_flags.p, 0, 2 * static_cast<size_t>(P) * sizeof(unsigned int),
                             ctx->stream));
    link_local_p2p(rks, static_cast<unsigned int*>(p2p_flags.p));
    op.p2p = true;
  }
  op.p2p_wait = [&](cudaStream_t s) -> int {
    if (p2p_seq == 0) return HJB_OK;  // V_0's halos came with the initial exchange
    for (int r = 0; r < P; ++r)
      for (int sd = 0; sd < 2; ++sd)
        if (rks[r].p2p.own_flag[sd]) {
          int e = wait_epoch(rks[r].p2p.own_flag[sd], p2p_seq, s);
          if (e) return e;
        }
    return HJB_OK;
  };
  op.sweep = [&](int k, int q, int mode, bool pp, cudaStream_t s) -> int {
    if (op.p2p)
      for (int r = 0; r < P; ++r) rks[r].p2p.epoch = p2p_seq + 1;
    for (int r = 0; r < P; ++r) {
      if (mode == kBnd && !rks[r].sp.bnd) continue;
      if (mode == kInner && !rks[r].sp.inner) continue;
      // kBoth: ranks without a boundary (P == 1) run their interior
      const int m = (mode == kBoth && !rks[r].sp.bnd) ? kInner : mode;
      unsigned long long* acc = pp ? &rs.st[r]->maxdv_slot[k & 1] : &rs.st[r]->maxdv_bits;
      CUDA_TRY(rks[r].launch(k, q, m, acc, s));
      ++per_pos;
    }
    if (op.p2p) ++p2p_seq;
    return HJB_OK;
  };
  op.exchange = [&](int k, int q, cudaStream_t s) -> int {
    for (int r = 0; r < P; ++r) xb[r] = rks[r].stage_out(k, q);
    return local_exchange(rks, xb, s);
  };
  // peer-store transport: the residual all-reduce through the ranks'
  // mailboxes as well (every contribution first: the ranks share a stream)
  DevBuf mbox_buf;
  unsigned int res_seq = 0;
  MboxSet mset;
  std::memset(&mset, 0, sizeof mset);
  if (op.p2p) {
    CUDA_TRY(mbox_buf.ensure(static_cast<size_t>(P) * sizeof(P2PMbox)));
    CUDA_TRY(cudaMemsetAsync(mbox_buf.p, 0, static_cast<size_t>(P) * sizeof(P2PMbox), ctx->stream));
    mset.n = P;
    for (int q = 0; q < P; ++q) mset.m[q] = static_cast<P2PMbox*>(mbox_buf.p) + q;
  }
  op.finish = [&](int k, bool pp, cudaGraphConditionalHandle hd, int use, cudaStream_t s) -> int {
    if (op.p2p) {
      const int sl = pp ? (k & 1) : -1;
      for (int r = 0; r < P; ++r) k_p2p_contribute<<<1, 32, 0, s>>>(rs.st[r], sl, mset, res_seq);
      CUDA_TRY(cudaGetLastError());
      const unsigned int need = static_cast<unsigned int>(P) * (res_seq / kMboxSlots + 1u);
      for (int r = 0; r < P; ++r) {
        int e = wait_epoch(&mset.m[r]->count[res_seq % kMboxSlots], need, s);
        if (e) return e;
        k_p2p_take<<<1, 32, 0, s>>>(mset.m[r], rs.st[r], sl, res_seq);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(launch_epilogue(rs.st[r], hd, use, s, pp ? &rs.st[r]->maxdv_slot[k & 1] : nullptr));
      }
      ++res_seq;
      per_pos += 3 * P;
      return HJB_OK;
    }
    k_reduce_ranks<<<1, 32, 0, s>>>(rs, pp ? (k & 1) : -1);
    CUDA_TRY(cudaGetLastError());
    for (int r = 0; r < P; ++r)
      CUDA_TRY(launch_epilogue(rs.st[r], hd, use, s, pp ? &rs.st[r]->maxdv_slot[k & 1] : nullptr));
    per_pos += 1 + P;
    return HJB_OK;
  };
  auto step = [&](int k, cudaGraphConditionalHandle hd, int use) -> int {
    per_pos = 0;
    return run_position(ls, ctx->stream, op, k, overlap, pipe, hd, use);
  };
  CUDA_TRY(cudaEventRecord(ls.e0, ctx->stream));
  // stream memory operations stay out of graph capture: the signalling
  // protocol runs the host-driven loop (as the NCCL transport always does)
  if ((rc = (op.signal || op.p2p) ? run_eager_loop(ctx, body, step)
                                   : run_sharded_loop(ctx, body, step)))
    return rc;
  CUDA_TRY(cudaEventRecord(ls.e1, ctx->stream));
  CUDA_TRY(cudaEventSynchronize(ls.e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ls.e0, ls.e1);
  if ((rc = fill_result(ctx, ms, res))) return rc;
  res->kernel = rks[0].ho ? HJB_KERNEL_HO4D : HJB_KERNEL_FAST4D;
  ctx->launches += per_pos * (res->iterations + body);
  const LoopState& st = *ctx->st_host;
  for (int r = 0; r < P; ++r) {
    if ((rc = unpad_rank(rks[r], p, st.iter, value_out + rks[r].geo.gbeg * s0, ctx->stream)))
      return rc;
    ++ctx->launches;
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (st.status == HJB_ERR_DIVERGED)
    return set_err(HJB_ERR_DIVERGED, "solve: diverging (residual grew 10x above its minimum)");
  return HJB_OK;
}

}  // extern "C"
