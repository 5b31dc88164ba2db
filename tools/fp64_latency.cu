// DFMA latency / low-occupancy throughput microbenchmark (B200, one CTA on one SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void chain(double* out, long long* cyc, int iters) {
  double a[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 0.9999999;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) a[i] = fma(a[i], b, c);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += a[i];
  if (s == 1.2345) out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 8);
  cudaMallocManaged(&cyc, 64 * 8);
  const int iters = 4096;
  for (int warps : {1, 2, 4, 8, 16}) {
#define RUN(C)                                                                          \
    chain<C><<<1, 32 * warps>>>(out, cyc, iters);                                       \
    cudaDeviceSynchronize();                                                            \
    printf("warps=%2d chains=%d: %.2f cycles/iter/warp -> %.1f DFMA/clk/SM\n", warps, C, \
           (double)cyc[0] / iters, 32.0 * warps * C * iters / cyc[0]);
    RUN(1) RUN(4) RUN(8)
  }
  return 0;
}
