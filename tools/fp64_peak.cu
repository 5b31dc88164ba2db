// FP64 peak microbenchmark for the roofline denominator (MEASURED_PEAKS.json has none).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
// Prints JSON: DFMA (FP64 pipe) and DMMA (mma.sync m8n8k4 f64, SASS DMMA.8x8x4) TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(acc[i][0]), "+d"(acc[i][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  float best_fma = 1e30f, best_mma = 1e30f;
  const int it_fma = 20000, it_mma = 20000;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, it_fma);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_fma) best_fma = ms;
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, it_mma);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_mma) best_mma = ms;
  }
  const double fma_flops = 2.0 * 8 * (double)it_fma * blocks * threads;
  // one m8n8k4 per warp = 8*8*4 MACs = 512 flops; 4 per iteration per warp
  const double mma_flops = 512.0 * 4 * (double)it_mma * blocks * (threads / 32);
  printf("{\"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f}\n", sms, fma_flops / best_fma / 1e9,
         mma_flops / best_mma / 1e9);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    fprintf(stderr, "%s\n", cudaGetErrorString(err));
    return 1;
  }
  return 0;
}
