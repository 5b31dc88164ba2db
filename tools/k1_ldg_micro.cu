// Streaming K1 matvec microbenchmark at sweep-stage scale: G CTAs (default 128), each a chain of
// `steps` dependent steps y = A_k x (A_k: w x w complex, column-major, padded to w4 columns), x <- f(y).
// The blocks of 4 "cells" (steps/2 blocks each) live in global memory; CTA i walks cell i % 4.
// MODE 0: register-direct: warp wp owns columns j = wp + 8 t; lane owns rows lane + 32 r; the loads
//         of step s+1 for a column are issued right after step s consumed that column (one step of
//         prefetch in registers); 8 warps; partial sums per warp reduced through shared memory.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 ldg_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
template <int NC, int RW, int CPW, int MODE>
__global__ void __launch_bounds__(256, 1) k_reg(const double2* __restrict__ S, double2* out, long long* cyc, int w,
                                                int steps, int nblk) {
  __shared__ double2 cur[128 * NC];
  __shared__ double2 red[8][72 * NC];
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int w4 = (w + 3) & ~3;
  const double2* base = S + (size_t)(blockIdx.x % 4) * nblk * w * w4;
  for (int i = tid; i < 128 * NC; i += 256) cur[i] = make_double2(i < w * NC ? 1e-2 : 0.0, 0.0);
  double2 buf[CPW][RW];
  // unconditional loads: columns >= w are zero padding (or the next block, multiplied by cur = 0),
  // rows >= w belong to the next column and are discarded; the pool has slack at its end
  const size_t bstride = (size_t)w * w4;
  const double2* colp = base + (size_t)wp * w + lane;  // column wp of block 0
  auto issue = [&](int s, int t) {
    const double2* col = colp + (size_t)(s % nblk) * bstride + (size_t)(8 * t) * w;
#pragma unroll
    for (int r = 0; r < RW; ++r) buf[t][r] = ldg_stream(col + 32 * r);
  };
#pragma unroll
  for (int t = 0; t < CPW; ++t) issue(0, t);
  __syncthreads();
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    double2 acc[RW][NC];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int q = 0; q < NC; ++q) acc[r][q] = make_double2(0, 0);
#pragma unroll
    for (int t = 0; t < CPW; ++t) {
      const int j = wp + 8 * t;
      double2 tv[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) tv[q] = cur[j * NC + q];
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          if (MODE == 2) { acc[r][q].x += buf[t][r].x; acc[r][q].y += tv[q].y; }
          else cfma(acc[r][q], buf[t][r], tv[q]);
        }
      if (MODE == 0 && s + 1 < steps) issue(s + 1, t);
    }
#pragma unroll
    for (int r = 0; r < RW; ++r)
      if (lane + 32 * r < w)
#pragma unroll
        for (int q = 0; q < NC; ++q) red[wp][(lane + 32 * r) * NC + q] = acc[r][q];
    __syncthreads();
    for (int e = tid; e < w * NC; e += 256) {
      double2 y = red[0][e];
#pragma unroll
      for (int g = 1; g < 8; ++g) { y.x += red[g][e].x; y.y += red[g][e].y; }
      cur[e] = make_double2(y.x * 1e-2, y.y * 1e-2);  // entries >= w*NC stay zero
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = cur[0]; }
}
template <int NC, int RW, int CPW, int MODE>
void run(int grid, int w) {
  const int nblk = 61, steps = 122, w4 = (w + 3) & ~3;
  double2* S; double2* out; long long* cyc;
  cudaMalloc(&S, sizeof(double2) * (4 * nblk * w * w4 + 65536));
  cudaMemset(S, 0, sizeof(double2) * (4 * nblk * w * w4 + 65536));
  cudaMalloc(&out, sizeof(double2) * grid); cudaMallocManaged(&cyc, sizeof(long long) * grid);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_reg<NC, RW, CPW, MODE><<<grid, 256>>>(S, out, cyc, w, steps, nblk);
  cudaEventRecord(a);
  k_reg<NC, RW, CPW, MODE><<<grid, 256>>>(S, out, cyc, w, steps, nblk);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long mx = 0; for (int i = 0; i < grid; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
  printf("mode %d NC=%d grid=%d w=%d: %.1f us, %.0f cycles/step (max CTA) (%s)\n", MODE, NC, grid, w, ms * 1e3,
         (double)mx / steps, cudaGetErrorString(e));
  cudaFree(S); cudaFree(out); cudaFree(cyc);
}
int main() {
  run<1, 3, 9, 0>(128, 70);
  run<1, 3, 9, 1>(128, 70);
  run<1, 3, 9, 2>(128, 70);
  run<2, 3, 9, 0>(64, 70);
  run<2, 3, 9, 1>(64, 70);
  return 0;
}
