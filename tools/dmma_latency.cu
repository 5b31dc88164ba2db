// DMMA (mma.sync m8n8k4 f64) latency / throughput vs independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8192); cudaMallocManaged(&cyc, 64);
  const int iters = 2000;
  for (int warps : {1, 4, 8}) {
#define R(CH) k<CH><<<1, 32 * warps>>>(out, cyc, iters); cudaDeviceSynchronize(); \
    printf("warps=%d chains=%d: %.1f cycles per DMMA per warp -> %.2f DMMA/clk/SM (peak ~0.25)\n", warps, CH, \
           (double)cyc[0] / (iters * CH), (double)warps * iters * CH / cyc[0]);
    R(1) R(2) R(4) R(8) R(16)
  }
}
