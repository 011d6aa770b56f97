// hjb_common.cuh — host-side plumbing shared by the C-ABI translation units:
// error state, device buffers and the context object.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "../../include/hjb.h"
#include "hjb_device.cuh"

namespace hjb {

extern thread_local std::string g_err;

inline int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return ::hjb::set_err(HJB_ERR_CUDA,                                               \
                            std::string(#expr " failed: ") + cudaGetErrorString(e_));   \
  } while (0)

// Grow-only device allocation.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  double* d() const { return static_cast<double*>(p); }
};

}  // namespace hjb

struct hjb_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  hjb::DevBuf v0, v1, v2, v3, cbuf, pcbuf, dbbuf, tables, scratch, hist, whist, xbuf;
  hjb::DevBuf gpa, gpb, gpc;  // GP bounds: k*, factor, per-point tables
  hjb::DevBuf pvtab;          // 4D fast path with axis-0-varying bounds: tables
  hjb::DevBuf pnbuf;          // 4D fast path with per-node bounds: padded lo / hi
  hjb::DevBuf cplane;         // constraint varying along axis 0 only: c per plane
  hjb::DevBuf tgbuf;          // target set: padded copy for the 4D fast path
  hjb::DevBuf tgx;            // target set: device copy of a host field
  hjb::LoopState* st = nullptr;
  hjb::LoopState* st_host = nullptr;  // pinned mirror
  long long launches = 0;
};
