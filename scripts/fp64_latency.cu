// Microbenchmark (B200): dependent FP64 latency and DFMA throughput per SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_latency scripts/fp64_latency.cu
// Measured: DADD/DFMA chain 8.1 cyc/op, FFMA 4.1, DFMA throughput 63 /clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a + threadIdx.x;
  float xf = (float)x;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 100; ++i) {
    #pragma unroll
    for (int u = 0; u < 64; ++u) {
      if (MODE == 0) x = x + b;
      if (MODE == 1) x = __fma_rn(x, a, b);
      if (MODE == 2) xf = __fmaf_rn(xf, (float)a, (float)b);
      if (MODE == 3) x = __shfl_sync(0xffffffffu, x, u & 31);
      if (MODE == 4) x = (x > b) ? x : b + 1.0;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + xf;
  if (threadIdx.x == 0) cyc[MODE] = (t1 - t0);
}
// throughput: many independent chains per thread, many warps
__global__ void kt(double* out, long long* cyc, double a, double b) {
  double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4=x0+4,x5=x0+5,x6=x0+6,x7=x0+7;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
    x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0);
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMallocManaged(&c, 64);
  const char* nm[] = {"DADD chain", "DFMA chain", "FFMA chain", "SHFL.f64 chain", "DSETP+sel chain"};
#define RUN(M) k<M><<<1, 32>>>(o, c, 1.0000001, 1e-9); cudaDeviceSynchronize(); k<M><<<1, 32>>>(o, c, 1.0000001, 1e-9); cudaDeviceSynchronize(); printf("%s: %.1f cyc/op\n", nm[M], c[M] / 6400.0);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4)
  for (int w : {1, 4, 8, 16, 32}) {
    kt<<<148, 32 * w>>>(o, c, 1.0000001, 1e-9); cudaDeviceSynchronize();
    kt<<<148, 32 * w>>>(o, c, 1.0000001, 1e-9); cudaDeviceSynchronize();
    printf("DFMA x8 indep, %d warps/SM: %.1f cyc per 8 ops per warp -> %.2f DFMA/clk/SM\n", w, c[0] / 1000.0, 8.0 * 32 * w / (c[0] / 1000.0));
  }
}
