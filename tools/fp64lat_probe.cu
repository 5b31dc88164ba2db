#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void lat(double* out, long long* cyc, int n, double a, double b) {
  double acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH> void run(int warps) {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 64);
  const int n = 4096;
  lat<CH><<<1, 32 * warps>>>(out, cyc, n, 0.999, 1e-3);
  cudaDeviceSynchronize();
  double c = (double)cyc[0] / n;  // cycles per iteration (CH dependent-chain steps per warp)
  printf("warps=%d chains=%d: %.2f cycles/iter -> %.2f cycles per DFMA latency-step, %.1f DFMA lanes/clk/SM\n", warps, CH, c, c,
         32.0 * warps * CH / c);
}
int main() {
  run<1>(1); run<4>(1); run<8>(1); run<4>(4); run<8>(4); run<4>(8); run<8>(8); run<2>(8); run<4>(7); run<16>(4);
}
