#include <cstdio>
#include <cuda_runtime.h>
template <int U, int WARPS>
__global__ void k(double* out, long long* cyc, int iters) {
  extern __shared__ double2 sm[];
  const int n = 8192;  // 128 KB
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_double2(i, 1);
  __syncthreads();
  double acc[U];
  for (int u = 0; u < U; ++u) acc[u] = 0;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int b = ((it * WARPS + wp) * U * 32) & (n - 1);
#pragma unroll
    for (int u = 0; u < U; ++u) { const double2 v = sm[(b + u * 32 + lane) & (n - 1)]; acc[u] += v.x; }
  }
  long long t1 = clock64();
  double s = 0; for (int u = 0; u < U; ++u) s += acc[u];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int U, int WARPS> void run() {
  double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMallocManaged(&cyc, 64);
  cudaFuncSetAttribute(k<U, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int iters = 2000;
  k<U, WARPS><<<1, 32 * WARPS, 131072>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  const double bytes = (double)iters * WARPS * U * 512;
  printf("U=%d warps=%d: %.1f B/clk (LDS.128)\n", U, WARPS, bytes / cyc[0]);
}
int main() { run<1, 7>(); run<4, 7>(); run<8, 7>(); run<16, 7>(); run<8, 16>(); run<4, 32>(); }
