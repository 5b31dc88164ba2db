// Microbenchmark of the K1 DFMA step (NC = 1, 2, 4) on one SM, data resident in shared memory:
// bar -> y = A cur (thread = (column group, row), columns unrolled by U) -> partials -> bar ->
// reduce partials into cur.  224 consumer threads, w = 70, 122 steps (one half chain of cfg2).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ void nbar() { asm volatile("bar.sync 1, 224;" ::: "memory"); }
template <int NC, int U, int MODE>
__global__ void __launch_bounds__(256, 1) bench(double2* out, long long* cyc, int w, int steps) {
  extern __shared__ double2 sm[];
  double2* A = sm;                  // w*w column-major
  double2* cur = A + w * w + 64;    // w*NC
  double2* red = cur + 128 * NC;    // 224*NC
  const int tid = threadIdx.x;
  for (int i = tid; i < w * w; i += blockDim.x) A[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  for (int i = tid; i < 128 * NC; i += blockDim.x) cur[i] = make_double2(1.0, 0.5);
  __syncthreads();
  if (tid >= 224) return;
  const int ngr = 224 / w, g = tid / w, i = tid - g * w;
  const bool act = g < ngr;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    double2 acc0[NC], acc1[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) acc0[q] = acc1[q] = make_double2(0, 0);
    if (act && MODE != 2) {
      for (int ch = 0; ch < 2; ++ch) {
        const int c0 = ch * 40, cw = min(40, w - c0);
        const int j1 = (g + 1) * cw / ngr;
        int jj = g * cw / ngr;
        const double2* col = A + c0 * w + i;
        if (MODE == 3) {  // loads only
          for (; jj < j1; ++jj) { const double2 a = col[jj * w]; acc0[0].x += a.x; acc1[0].y += a.y; }
        }
        if (MODE == 4) {  // DFMA only (operands in registers)
          const double2 a = make_double2(1e-3 * i, 2e-3), tvv = make_double2(0.5, 0.25);
          for (; jj + 4 <= j1; jj += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int q = 0; q < NC; ++q) cfma((u & 1) ? acc1[q] : acc0[q], a, tvv);
          }
        }
        if (MODE == 0) {
          for (; jj + U <= j1; jj += U) {
            double2 a[U], tv[U][NC];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              a[u] = col[(jj + u) * w];
#pragma unroll
              for (int q = 0; q < NC; ++q) tv[u][q] = cur[(c0 + jj + u) * NC + q];
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int q = 0; q < NC; ++q) cfma((u & 1) ? acc1[q] : acc0[q], a[u], tv[u][q]);
          }
        }
        for (; jj < j1; ++jj) {
          const double2 a = col[jj * w];
#pragma unroll
          for (int q = 0; q < NC; ++q) cfma(acc0[q], a, cur[(c0 + jj) * NC + q]);
        }
      }
#pragma unroll
      for (int q = 0; q < NC; ++q) red[(g * w + i) * NC + q] = make_double2(acc0[q].x + acc1[q].x, acc0[q].y + acc1[q].y);
    }
    nbar();
    for (int e = tid; e < w * NC; e += 224) {
      const int ii = e / NC, q = e - ii * NC;
      double2 y = red[ii * NC + q];
      for (int gg = 1; gg < ngr; ++gg) { const double2 v = red[(gg * w + ii) * NC + q]; y.x += v.x; y.y += v.y; }
      cur[e] = make_double2(y.x * 1e-3, y.y * 1e-3);
    }
    nbar();
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; out[0] = cur[0]; }
}
template <int NC, int U, int MODE>
void run(const char* name, int w) {
  double2* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMallocManaged(&cyc, 64);
  const int steps = 122;
  const size_t smem = (size_t)(w * w + 64 + 128 * NC + 224 * NC) * 16;
  cudaFuncSetAttribute(bench<NC, U, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench<NC, U, MODE><<<1, 256, smem>>>(out, cyc, w, steps);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%-28s w=%d NC=%d U=%d: %.0f cycles/step (%s)\n", name, w, NC, U, (double)cyc[0] / steps, cudaGetErrorString(e));
}
int main() {
  run<1, 1, 2>("bars + epilogue only", 70);
  run<1, 1, 3>("loads only", 70);
  run<1, 4, 4>("dfma only", 70);
  run<4, 4, 4>("dfma only", 70);
  run<1, 1, 1>("no unroll", 70);
  run<1, 4, 0>("unroll 4", 70);
  run<1, 8, 0>("unroll 8", 70);
  run<2, 4, 0>("unroll 4", 70);
  run<4, 4, 0>("unroll 4", 70);
  run<4, 2, 0>("unroll 2", 70);

  return 0;
}
