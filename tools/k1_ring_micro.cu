// K1 DFMA-path microbenchmark at sweep scale: G CTAs, each 7 consumer warps + 1 producer warp; the
// producer streams w x w4 complex blocks (4 cells x 61 blocks in global memory) through an NS-slot
// shared-memory ring in chunks of 7*JW columns (cp.async.bulk + mbarriers); consumers: lanes own rows
// lane + 32 r, warp wp owns columns wp*JW.. of each chunk; per step: partials -> bar -> reduce -> bar.
//   PRED: predicate the row-block loads on row < w (fewer shared-memory wavefronts for the tail block)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1510_01831_b200/csrc/pt_device.cuh"

template <int NC, int RW, int JW, int NSL, int PRED, int MODE = 0>
__global__ void __launch_bounds__(256, 1) kern(const double2* __restrict__ S, double2* out, long long* cyc, int w,
                                               int steps, int nblk) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int JC = 7 * JW;
  const int w4 = (w + 3) & ~3;
  const int slot_bytes = ((JC * w * 16) + 127) & ~127;
  unsigned char* ring = smem;
  double2* cur = reinterpret_cast<double2*>(ring + NSL * slot_bytes);
  double2* red = cur + 128 * NC;
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 7 * 128 * NC);
  uint64_t* lempty = full + NSL;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int nch = (w4 + JC - 1) / JC, total = steps * nch;
  const double2* base = S + (size_t)(blockIdx.x % 4) * nblk * w * w4;
  for (int i = tid; i < 128 * NC; i += blockDim.x) cur[i] = make_double2(i < w * NC ? 1e-2 : 0.0, 0.0);
  if (tid == 0) {
    for (int s = 0; s < NSL; ++s) { mbar_init(&full[s], 1); mbar_init(&lempty[s], 7); }
    fence_mbar_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (wp == 7) {
    if (lane == 0 && MODE != 2) {
      int slot = 0; uint32_t ph = 0;
      for (int c = 0; c < total; ++c) {
        if (c >= NSL) mbar_wait(&lempty[slot], ph ^ 1);
        const int s = c / nch, ch = c - s * nch, c0 = ch * JC, cw = min(JC, w4 - c0);
        const uint32_t bytes = cw * w * 16;
        mbar_expect_tx(&full[slot], bytes);
        bulk_g2s(ring + slot * slot_bytes, base + (size_t)(s % nblk) * w * w4 + (size_t)c0 * w, bytes, &full[slot]);
        if (++slot == NSL) { slot = 0; ph ^= 1; }
      }
    }
  } else {
    int slot = 0; uint32_t ph = 0;
    for (int s = 0; s < steps; ++s) {
      double2 acc[RW][NC], acc2[RW][NC];
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[r][q] = acc2[r][q] = make_double2(0, 0);
      for (int ch = 0; ch < nch; ++ch) {
        if (MODE != 2 && MODE < 5) mbar_wait(&full[slot], ph);
        const double2* blk = reinterpret_cast<const double2*>(ring + slot * slot_bytes);
        const int c0 = ch * JC, cw = min(JC, w - c0);
        if (MODE == 3 || MODE == 4) {
          // all loads of the warp's JW columns first, then the FMAs; two accumulator sets (MODE 4)
          double2 av[JW][RW], tvv[JW][NC];
#pragma unroll
          for (int u = 0; u < JW; ++u) {
            const int jj = wp * JW + u;
            const bool ok = jj < cw;
#pragma unroll
            for (int q = 0; q < NC; ++q) tvv[u][q] = ok ? cur[(c0 + jj) * NC + q] : make_double2(0, 0);
            const double2* col = blk + jj * w + lane;
#pragma unroll
            for (int r = 0; r < RW; ++r)
              av[u][r] = (ok && (r + 1 < RW || lane + 32 * r < w)) ? col[32 * r] : make_double2(0, 0);
          }
#pragma unroll
          for (int u = 0; u < JW; ++u)
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
              for (int q = 0; q < NC; ++q) cfma((MODE == 4 && (u & 1)) ? acc2[r][q] : acc[r][q], av[u][r], tvv[u][q]);
        } else
#pragma unroll
        for (int u = 0; u < JW; ++u) {
          const int jj = wp * JW + u;
          if (MODE != 1 && jj < cw) {
            double2 tv[NC];
#pragma unroll
            for (int q = 0; q < NC; ++q) tv[q] = cur[(c0 + jj) * NC + q];
            const double2* col = blk + jj * w + lane;
#pragma unroll
            for (int r = 0; r < RW; ++r) {
              double2 a = make_double2(0, 0);
              if (!PRED || r + 1 < RW || lane + 32 * r < w) a = col[32 * r];
#pragma unroll
              for (int q = 0; q < NC; ++q) cfma(acc[r][q], a, tv[q]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_relaxed(&lempty[slot]);
        if (++slot == NSL) { slot = 0; ph ^= 1; }
      }
#pragma unroll
      for (int r = 0; r < RW; ++r)
        if (lane + 32 * r < w)
#pragma unroll
          for (int q = 0; q < NC; ++q) red[(wp * 128 + lane + 32 * r) * NC + q] = cadd(acc[r][q], acc2[r][q]);
      named_bar(1, 224);
      for (int e = tid; e < w * NC; e += 224) {
        double2 y = red[e];
#pragma unroll
        for (int g = 1; g < 7; ++g) y = cadd(y, red[g * 128 * NC + e]);
        cur[e] = make_double2(y.x * 1e-2, y.y * 1e-2);
      }
      named_bar(1, 224);
    }
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = cur[0]; }
}
template <int NC, int RW, int JW, int NSL, int PRED, int MODE = 0>
void run(int grid, int w) {
  const int nblk = 61, steps = 122, w4 = (w + 3) & ~3;
  double2* S; double2* out; long long* cyc;
  cudaMalloc(&S, sizeof(double2) * (4 * nblk * w * w4 + 65536));
  cudaMemset(S, 0, sizeof(double2) * (4 * nblk * w * w4 + 65536));
  cudaMalloc(&out, sizeof(double2) * grid); cudaMallocManaged(&cyc, sizeof(long long) * grid);
  const int slot_bytes = ((7 * JW * w * 16) + 127) & ~127;
  const size_t smem = (size_t)NSL * slot_bytes + (128 * NC + 7 * 128 * NC) * 16 + 2 * NSL * 8 + 64;
  cudaFuncSetAttribute(kern<NC, RW, JW, NSL, PRED, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  kern<NC, RW, JW, NSL, PRED, MODE><<<grid, 256, smem>>>(S, out, cyc, w, steps, nblk);
  cudaEventRecord(a);
  kern<NC, RW, JW, NSL, PRED, MODE><<<grid, 256, smem>>>(S, out, cyc, w, steps, nblk);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long mx = 0; for (int i = 0; i < grid; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
  printf("mode=%d NC=%d JW=%d NS=%d pred=%d grid=%d w=%d smem=%zuKB: %.1f us, %.0f cycles/step (%s)\n", MODE, NC, JW, NSL, PRED,
         grid, w, smem >> 10, ms * 1e3, (double)mx / steps, cudaGetErrorString(e));
  cudaFree(S); cudaFree(out); cudaFree(cyc);
}
int main() {
  run<1, 3, 2, 8, 1, 2>(128, 70);
  run<1, 3, 5, 5, 1, 2>(128, 70);
  run<1, 3, 2, 8, 1, 3>(128, 70);
  run<1, 3, 5, 5, 1, 3>(128, 70);
  run<1, 3, 2, 8, 1, 4>(128, 70);
  run<1, 3, 5, 5, 1, 4>(128, 70);
  run<2, 3, 5, 5, 1, 4>(64, 70);
  run<4, 3, 2, 8, 1, 4>(32, 70);
  return 0;
}
