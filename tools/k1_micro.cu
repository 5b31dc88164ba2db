// Microbenchmark of the K1 matvec step on one SM: y = A x, A w x w complex column-major in shared
// memory, x [w][NC]; 7 warps.  MODE 1: DFMA, lanes own rows, warps stride columns.  MODE 2: same
// with x in registers (no x loads).  MODE 3: DMMA m8n8k4 (NC padded to 8): warps own (8-row tile,
// K half) units; Cr += Ar*Br + (-Ai)*Bi, Ci += Ar*Bi + Ai*Br.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int NC, int MODE>
__global__ void bench(double2* out, long long* cyc, int w, int steps) {
  extern __shared__ double2 sm[];
  double2* A = sm;                 // w*w (+ padding)
  double2* X = A + w * w + 1024;   // w*NC (padded to 8 cols for MODE 3)
  double2* R = X + 136 * 8;        // partials (7*w*8 max)
  for (int i = threadIdx.x; i < w * w + 1024; i += blockDim.x) A[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  for (int i = threadIdx.x; i < 136 * 8; i += blockDim.x) X[i] = make_double2(1.0, 0.5);
  __syncthreads();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, rw = (w + 31) >> 5;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    if (MODE == 6) {
      // rows split across warps: warp = (row block rb of 32, column half hf); 2 interleaved accs
      const int nrb = rw, nh = 2;
      if (wp < nrb * nh) {
        const int rb = wp % nrb, hf = wp / nrb;
        const int i = rb * 32 + lane;
        const int j0 = hf * ((w + 1) / 2), j1 = hf == 0 ? (w + 1) / 2 : w;
        double2 acc[NC], acc2[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[q] = acc2[q] = make_double2(0, 0);
        const double2* col = A + i;
        int j = j0;
#pragma unroll 4
        for (; j + 1 < j1; j += 2) {
          const double2 a0 = col[j * w], a1 = col[(j + 1) * w];
#pragma unroll
          for (int q = 0; q < NC; ++q) { cfma(acc[q], a0, X[j * NC + q]); cfma(acc2[q], a1, X[(j + 1) * NC + q]); }
        }
        if (j < j1) {
          const double2 a0 = col[j * w];
#pragma unroll
          for (int q = 0; q < NC; ++q) cfma(acc[q], a0, X[j * NC + q]);
        }
        if (i < w)
#pragma unroll
          for (int q = 0; q < NC; ++q) { double2 v = acc[q]; v.x += acc2[q].x; v.y += acc2[q].y; R[(hf * w + i) * NC + q] = v; }
      }
      asm volatile("bar.sync 1, 224;");
      for (int e = threadIdx.x; e < w * NC; e += 224) {
        const double2 y0 = R[e], y1 = R[w * NC + e];
        X[e] = make_double2((y0.x + y1.x) * 1e-3, (y0.y + y1.y) * 1e-3);
      }
      asm volatile("bar.sync 1, 224;");
    } else if (MODE == 4) {
      double2 acc[4][NC], acc2[4][NC];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[r][q] = acc2[r][q] = make_double2(0, 0);
      int jj = wp;
      for (; jj + 7 < w; jj += 14) {
        double2 tv[NC], tw[NC], a0[4], a1[4];
#pragma unroll
        for (int q = 0; q < NC; ++q) { tv[q] = X[jj * NC + q]; tw[q] = X[(jj + 7) * NC + q]; }
#pragma unroll
        for (int r = 0; r < 4; ++r) if (r < rw) { a0[r] = A[jj * w + lane + 32 * r]; a1[r] = A[(jj + 7) * w + lane + 32 * r]; }
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (r < rw) {
#pragma unroll
            for (int q = 0; q < NC; ++q) { cfma(acc[r][q], a0[r], tv[q]); cfma(acc2[r][q], a1[r], tw[q]); }
          }
      }
      if (jj < w) {
        double2 tv[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) tv[q] = X[jj * NC + q];
#pragma unroll
        for (int r = 0; r < 4; ++r) if (r < rw) { const double2 a = A[jj * w + lane + 32 * r];
#pragma unroll
          for (int q = 0; q < NC; ++q) cfma(acc[r][q], a, tv[q]); }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (lane + 32 * r < w)
#pragma unroll
          for (int q = 0; q < NC; ++q) { double2 v = acc[r][q]; v.x += acc2[r][q].x; v.y += acc2[r][q].y; R[(wp * w + lane + 32 * r) * NC + q] = v; }
      asm volatile("bar.sync 1, 224;");
      for (int e = threadIdx.x; e < w * NC; e += 224) {
        double2 y = R[e];
        for (int g = 1; g < 7; ++g) { double2 v = R[g * w * NC + e]; y.x += v.x; y.y += v.y; }
        X[e] = make_double2(y.x * 1e-3, y.y * 1e-3);
      }
      asm volatile("bar.sync 1, 224;");
    } else if (MODE == 5) {
      // DMMA, units = (pair of M tiles, K quarter): two independent accumulator pairs per warp
      const int nmt = (w + 7) / 8, nks = (w + 3) / 4, kq = (nks + 3) / 4;
      const int npair = (nmt + 1) / 2, units = npair * 4;
      const int ar = lane >> 2, ak = lane & 3;
      for (int u = wp; u < units; u += 7) {
        const int pr = u >> 2, qt = u & 3;
        const int m0 = 2 * pr, m1 = min(2 * pr + 1, nmt - 1);
        const int ks0 = qt * kq, ks1 = min(nks, ks0 + kq);
        double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int ks = ks0; ks < ks1; ++ks) {
          const int k = ks * 4 + ak;
          const double2 b = X[k * 8 + ar];
          const double2 a0 = A[k * w + m0 * 8 + ar];
          const double2 a1 = A[k * w + m1 * 8 + ar];
          dmma(c[0], c[1], a0.x, b.x);
          dmma(c[4], c[5], a1.x, b.x);
          dmma(c[2], c[3], a0.x, b.y);
          dmma(c[6], c[7], a1.x, b.y);
          dmma(c[0], c[1], -a0.y, b.y);
          dmma(c[4], c[5], -a1.y, b.y);
          dmma(c[2], c[3], a0.y, b.x);
          dmma(c[6], c[7], a1.y, b.x);
        }
        const int r0 = m0 * 8 + ar, r1 = m1 * 8 + ar;
        R[(qt * 136 + r0) * 8 + 2 * ak] = make_double2(c[0], c[2]);
        R[(qt * 136 + r0) * 8 + 2 * ak + 1] = make_double2(c[1], c[3]);
        if (m1 != m0) {
          R[(qt * 136 + r1) * 8 + 2 * ak] = make_double2(c[4], c[6]);
          R[(qt * 136 + r1) * 8 + 2 * ak + 1] = make_double2(c[5], c[7]);
        }
      }
      asm volatile("bar.sync 1, 224;");
      for (int e = threadIdx.x; e < w * 8; e += 224) {
        double2 y = R[e];
        for (int g = 1; g < 4; ++g) { double2 v = R[g * 136 * 8 + e]; y.x += v.x; y.y += v.y; }
        X[e] = make_double2(y.x * 1e-3, y.y * 1e-3);
      }
      asm volatile("bar.sync 1, 224;");
    } else if (MODE <= 2) {
      double2 acc[4][NC];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[r][q] = make_double2(0, 0);
      double2 tr[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) tr[q] = X[q];
      for (int jj = wp; jj < w; jj += 7) {
        double2 tv[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) tv[q] = MODE == 1 ? X[jj * NC + q] : tr[q];
        const double2* col = A + jj * w + lane;
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (r < rw) {
            const double2 a = col[32 * r];
#pragma unroll
            for (int q = 0; q < NC; ++q) cfma(acc[r][q], a, tv[q]);
          }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (lane + 32 * r < w)
#pragma unroll
          for (int q = 0; q < NC; ++q) R[(wp * w + lane + 32 * r) * NC + q] = acc[r][q];
      asm volatile("bar.sync 1, 224;");
      for (int e = threadIdx.x; e < w * NC; e += 224) {
        double2 y = R[e];
        for (int g = 1; g < 7; ++g) { double2 v = R[g * w * NC + e]; y.x += v.x; y.y += v.y; }
        X[e] = make_double2(y.x * 1e-3, y.y * 1e-3);
      }
      asm volatile("bar.sync 1, 224;");
    } else {
      // DMMA: M tiles of 8 rows (mt < ceil(w/8)), K steps of 4 (ks < ceil(w/4)), N = 8 columns
      const int nmt = (w + 7) / 8, nks = (w + 3) / 4, kh = (nks + 1) / 2;
      const int units = nmt * 2;
      const int ar = lane >> 2, ak = lane & 3;   // A frag: row ar, k ak ; B frag: k = ak, col = ar
      for (int u = wp; u < units; u += 7) {
        const int mt = u >> 1, half = u & 1;
        const int ks0 = half * kh, ks1 = min(nks, ks0 + kh);
        double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0;
        for (int ks = ks0; ks < ks1; ++ks) {
          const int k = ks * 4 + ak;
          const double2 a = A[k * w + mt * 8 + ar];
          const double2 b = X[k * 8 + ar];
          dmma(cr0, cr1, a.x, b.x);
          dmma(cr0, cr1, -a.y, b.y);
          dmma(ci0, ci1, a.x, b.y);
          dmma(ci0, ci1, a.y, b.x);
        }
        // C frag: row ar, cols 2*ak, 2*ak+1
        const int row = mt * 8 + ar;
        R[(half * 136 + row) * 8 + 2 * ak] = make_double2(cr0, ci0);
        R[(half * 136 + row) * 8 + 2 * ak + 1] = make_double2(cr1, ci1);
      }
      asm volatile("bar.sync 1, 224;");
      for (int e = threadIdx.x; e < w * 8; e += 224) {
        const double2 y0 = R[e], y1 = R[136 * 8 + e];
        X[e] = make_double2((y0.x + y1.x) * 1e-3, (y0.y + y1.y) * 1e-3);
      }
      asm volatile("bar.sync 1, 224;");
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (threadIdx.x == 0) out[blockIdx.x] = X[0];
}
int main() {
  double2* out; long long* cyc;
  cudaMalloc(&out, 1024 * 16); cudaMallocManaged(&cyc, 1024 * 8);
  const int steps = 200;
  for (int w : {70, 86}) {
#define RUN(NC, MODE)                                                                         \
  {                                                                                           \
    size_t smem = (w * w + 1024 + 136 * 8 + (7 * w * 8 > 4 * 136 * 8 ? 7 * w * 8 : 4 * 136 * 8)) * 16;                               \
    cudaFuncSetAttribute(bench<NC, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    bench<NC, MODE><<<1, 224, smem>>>(out, cyc, w, steps);                                    \
    cudaError_t e = cudaDeviceSynchronize();                                                  \
    printf("w=%d NC=%d mode=%d: %.0f cycles/step (%s) ideal_fma=%.0f\n", w, NC, MODE,         \
           (double)cyc[0] / steps, cudaGetErrorString(e), 4.0 * w * w * NC / 64);             \
  }
    RUN(1, 1) RUN(1, 6) RUN(2, 1) RUN(2, 6) RUN(4, 1) RUN(4, 6) RUN(8, 5)
  }
  return 0;
}
