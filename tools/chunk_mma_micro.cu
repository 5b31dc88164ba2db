// DMMA issue patterns for the complex tile product (8 warps per SM, operands in shared memory)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1510_01831_b200/csrc -o tools/chunk_mma_micro tools/chunk_mma_micro.cu
#include <cstdio>
#include "pt_device.cuh"

__device__ __forceinline__ void dmma4(double (&a)[8], double ar, double ai, double br, double bi) {
  dmma_f64(a[0], a[1], ar, br);
  dmma_f64(a[2], a[3], ai, bi);
  dmma_f64(a[4], a[5], ar, bi);
  dmma_f64(a[6], a[7], ai, br);
}

// mode 0: 1 pair, loads + dmul sg per k-step; 1: 1 pair, no dmul; 2: 2 pairs (2 B tiles) no dmul;
// 3: 4 pairs (2x2); 4: 1 pair, registers only (no loads); 5: 2x2 registers only
__global__ void k(int reps, int nks, int mode, unsigned long long* out, double* sink) {
  extern __shared__ __align__(128) double2 sm[];
  for (int i = threadIdx.x; i < 4 * 128 * 8; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  const int lane = threadIdx.x & 31, r8 = lane >> 2, kl = lane & 3, wp = threadIdx.x >> 5;
  const double2* A0 = sm + r8;
  const double2* B0 = sm + 2 * 128 * 8 + r8;
  double acc[4][8];
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 8; ++i) acc[j][i] = 0;
  const int ks0 = wp * nks, ks1 = ks0 + nks;
  const double sg = sink[1];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (mode <= 1) {
#pragma unroll 4
      for (int ks = ks0; ks < ks1; ++ks) {
        const int kk = (ks * 4 + kl) & 127;
        double2 a0 = A0[kk * 8];
        double2 b0 = B0[kk * 8];
        if (mode == 0) b0 = make_double2(b0.x * sg, b0.y * sg);
        dmma4(acc[0], a0.x, a0.y, b0.x, b0.y);
      }
    } else if (mode == 2) {
#pragma unroll 4
      for (int ks = ks0; ks < ks1; ++ks) {
        const int kk = (ks * 4 + kl) & 127;
        double2 a0 = A0[kk * 8];
        double2 b0 = B0[kk * 8], b1 = B0[(128 + kk) * 8];
        dmma4(acc[0], a0.x, a0.y, b0.x, b0.y);
        dmma4(acc[1], a0.x, a0.y, b1.x, b1.y);
      }
    } else if (mode == 3) {
#pragma unroll 2
      for (int ks = ks0; ks < ks1; ++ks) {
        const int kk = (ks * 4 + kl) & 127;
        double2 a0 = A0[kk * 8], a1 = A0[(128 + kk) * 8];
        double2 b0 = B0[kk * 8], b1 = B0[(128 + kk) * 8];
        dmma4(acc[0], a0.x, a0.y, b0.x, b0.y);
        dmma4(acc[1], a0.x, a0.y, b1.x, b1.y);
        dmma4(acc[2], a1.x, a1.y, b0.x, b0.y);
        dmma4(acc[3], a1.x, a1.y, b1.x, b1.y);
      }
    } else if (mode == 4) {
      double2 a0 = A0[kl * 8], b0 = B0[kl * 8];
#pragma unroll 4
      for (int ks = ks0; ks < ks1; ++ks) dmma4(acc[0], a0.x, a0.y, b0.x, b0.y);
    } else {
      double2 a0 = A0[kl * 8], b0 = B0[kl * 8], a1 = A0[(8 + kl) * 8], b1 = B0[(8 + kl) * 8];
#pragma unroll 2
      for (int ks = ks0; ks < ks1; ++ks) {
        dmma4(acc[0], a0.x, a0.y, b0.x, b0.y);
        dmma4(acc[1], a0.x, a0.y, b1.x, b1.y);
        dmma4(acc[2], a1.x, a1.y, b0.x, b0.y);
        dmma4(acc[3], a1.x, a1.y, b1.x, b1.y);
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  double s = 0;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 8; ++i) s += acc[j][i];
  if (s == 12345.0) sink[0] = s;
}

int main() {
  unsigned long long* d;
  double* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 16);
  double one[2] = {0, 1.0};
  cudaMemcpy(sink, one, 16, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  unsigned long long h[148];
  const int dm[6] = {4, 4, 8, 16, 4, 16};
  for (int mode = 0; mode < 6; ++mode)
    for (int nks : {4, 32}) {
      const int reps = 2000;
      k<<<148, 256, 80 * 1024>>>(reps, nks, mode, d, sink);
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      const double per = (double)h[0] / reps;
      printf("mode %d k-steps/warp %2d: %6.0f cycles per chunk (%.3f DMMA/clk/SM)  %s\n", mode, nks, per,
             8.0 * nks * dm[mode] / per, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
