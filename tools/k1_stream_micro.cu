// Streaming microbenchmark: one CTA = 7 consumer warps + 1 producer warp, w x w complex blocks
// streamed from global memory through an 8-slot shared-memory ring (cp.async.bulk + mbarriers),
// y = A x with DMMA (NC=8) per block, `steps` dependent steps.  Mirrors K1's loop structure.
//   MODE 0: full (producer + waits + DMMA)   MODE 1: data preloaded once, no producer/waits
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1510_01831_b200/csrc/pt_device.cuh"

#define NSLOT 8
#define JC 16
template <int MODE>
__global__ void __launch_bounds__(256, 1) kern(const double2* __restrict__ S, double2* out, long long* cyc, int w,
                                               int steps, int slot_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  double2* cur = reinterpret_cast<double2*>(ring + NSLOT * slot_bytes);
  double2* red = cur + 128 * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 7 * 72 * 8);
  uint64_t* lempty = full + NSLOT;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int w4 = (w + 3) & ~3, nch = (w4 + JC - 1) / JC, total = steps * nch;
  for (int i = tid; i < 128 * 8; i += blockDim.x) cur[i] = make_double2(i < w * 8 ? 1e-2 : 0.0, 0.0);
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) { mbar_init(&full[s], 1); mbar_init(&lempty[s], 7); }
    fence_mbar_init();
  }
  __syncthreads();
  if (MODE >= 1 && tid < 224)
    for (int i = tid; i < NSLOT * slot_bytes / 16; i += 224) reinterpret_cast<double2*>(ring)[i] = S[i % (w * w4)];
  __syncthreads();
  long long t0 = clock64();
  if (wp == 7) {
    if (lane == 0 && MODE == 0)
      for (int c = 0; c < total; ++c) {
        const int slot = c & 7, u = c >> 3, ch = c % nch, c0 = ch * JC, cw = min(JC, w4 - c0);
        if (u > 0) mbar_wait(&lempty[slot], (u - 1) & 1);
        const uint32_t bytes = cw * w * 16;
        mbar_expect_tx(&full[slot], bytes);
        bulk_g2s(ring + slot * slot_bytes, S + (size_t)((c / nch) % 60) * w * w4 + c0 * w, bytes, &full[slot]);
      }
  } else {
    const int nmt = (w + 7) >> 3, ar = lane >> 2, ak = lane & 3;
    int c = 0;
    if (MODE == 6) {
      // K split: warp wp takes k-steps ks = wp mod 7 (over the whole step), all row tiles (<= 9 here)
      for (int s = 0; s < steps; ++s) {
        double cc[9][4];
#pragma unroll
        for (int t = 0; t < 9; ++t) cc[t][0] = cc[t][1] = cc[t][2] = cc[t][3] = 0.0;
        const int nks = w4 >> 2;
        for (int ks = wp; ks < nks; ks += 7) {
          const int k = ks * 4 + ak;
          const double2* blk = reinterpret_cast<const double2*>(ring) + (size_t)k * w + ar;
          const double2 bv = cur[k * 8 + ar];
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            const double2 av = blk[t * 8];
            dmma_f64(cc[t][0], cc[t][1], av.x, bv.x);
            dmma_f64(cc[t][2], cc[t][3], av.x, bv.y);
            dmma_f64(cc[t][0], cc[t][1], -av.y, bv.y);
            dmma_f64(cc[t][2], cc[t][3], av.y, bv.x);
          }
        }
#pragma unroll
        for (int t = 0; t < 9; ++t) {
          const int row = t * 8 + ar;
          if (row < w) {
            red[(wp * 72 + row) * 8 + 2 * ak] = make_double2(cc[t][0], cc[t][2]);
            red[(wp * 72 + row) * 8 + 2 * ak + 1] = make_double2(cc[t][1], cc[t][3]);
          }
        }
        named_bar(1, 224);
        for (int e = tid; e < w * 8; e += 224) {
          double2 y = red[e];
          for (int g = 1; g < 7; ++g) { const double2 v = red[g * 72 * 8 + e]; y.x += v.x; y.y += v.y; }
          cur[e] = make_double2(y.x * 1e-3, y.y * 1e-3);
        }
        named_bar(1, 224);
      }
    } else
    for (int s = 0; s < steps; ++s) {
      double cm[3][4], cm2[3][4];
#pragma unroll
      for (int it = 0; it < 3; ++it)
        for (int z = 0; z < 4; ++z) cm[it][z] = cm2[it][z] = 0.0;
      for (int ch = 0; ch < nch; ++ch, ++c) {
        const int slot = c & 7;
        if (MODE == 0 || MODE == 4) mbar_wait(&full[slot], (c >> 3) & 1);
        const double2* blk = reinterpret_cast<const double2*>(ring + slot * slot_bytes);
        const int c0 = ch * JC, nks = min(JC, w4 - c0) >> 2;
        const double2* ap = blk + ak * w + ar;
        const double2* bp = cur + (c0 + ak) * 8 + ar;
        if (MODE >= 2) {
          double2 bf[JC / 4], af[JC / 4][3];
#pragma unroll
          for (int ks = 0; ks < JC / 4; ++ks) {
            bf[ks] = ks < nks ? bp[ks * 32] : make_double2(0, 0);
#pragma unroll
            for (int it = 0; it < 3; ++it) {
              const int mt = wp + 7 * it;
              af[ks][it] = (ks < nks && mt < nmt) ? ap[ks * 4 * w + mt * 8] : make_double2(0, 0);
            }
          }
#pragma unroll
          for (int ks = 0; ks < JC / 4; ++ks)
#pragma unroll
            for (int it = 0; it < 3; ++it) {
              const int mt = wp + 7 * it;
              if (mt < nmt) {
                double* cc = (MODE == 3 && (ks & 1)) ? cm2[it] : cm[it];
                dmma_f64(cc[0], cc[1], af[ks][it].x, bf[ks].x);
                dmma_f64(cc[2], cc[3], af[ks][it].x, bf[ks].y);
                dmma_f64(cc[0], cc[1], -af[ks][it].y, bf[ks].y);
                dmma_f64(cc[2], cc[3], af[ks][it].y, bf[ks].x);
              }
            }
        } else
#pragma unroll
        for (int ks = 0; ks < JC / 4; ++ks)
          if (ks < nks) {
            const double2 bv = bp[ks * 32];
#pragma unroll
            const double nbi = -bv.y;  // negation once per k-step, shared by the warp's tiles
            for (int it = 0; it < 3; ++it) {
              const int mt = wp + 7 * it;
              if (mt < nmt) {
                const double2 av = ap[ks * 4 * w + mt * 8];
                dmma_f64(cm[it][0], cm[it][1], av.x, bv.x);
                dmma_f64(cm[it][2], cm[it][3], av.x, bv.y);
                dmma_f64(cm[it][0], cm[it][1], av.y, MODE == 5 ? bv.y : nbi);
                dmma_f64(cm[it][2], cm[it][3], av.y, bv.x);
              }
            }
          }
        __syncwarp();
        if ((MODE == 0 || MODE == 4) && lane == 0) mbar_arrive(&lempty[slot]);
      }
#pragma unroll
      for (int it = 0; it < 3; ++it) {
        const int mt = wp + 7 * it, row = mt * 8 + ar;
        if (mt < nmt && row < w) {
          red[row * 8 + 2 * ak] = make_double2((cm[it][0] + cm2[it][0]) * 1e-3, (cm[it][2] + cm2[it][2]) * 1e-3);
          red[row * 8 + 2 * ak + 1] = make_double2((cm[it][1] + cm2[it][1]) * 1e-3, (cm[it][3] + cm2[it][3]) * 1e-3);
        }
      }
      named_bar(1, 224);
      for (int e = tid; e < w * 8; e += 224) cur[e] = red[e];
      named_bar(1, 224);
    }
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; out[0] = cur[0]; }
}
int main() {
  const int w = 70, w4 = 72, steps = 61;
  double2* S;
  cudaMalloc(&S, sizeof(double2) * 60 * w * w4);
  cudaMemset(S, 0, sizeof(double2) * 60 * w * w4);
  double2* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMallocManaged(&cyc, 64);
  const int slot = JC * w * 16;
  const size_t smem = NSLOT * slot + (128 * 8 + 7 * 72 * 8) * 16 + 2 * NSLOT * 8 + 64;
  cudaFuncSetAttribute(kern<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#define RUNM(M, NAME)                                                                       \
  {                                                                                         \
    cudaFuncSetAttribute(kern<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kern<M><<<1, 256, smem>>>(S, out, cyc, w, steps, slot);                                 \
    cudaError_t e = cudaDeviceSynchronize();                                                \
    printf("%-44s %.0f cycles/step (%s)\n", NAME, (double)cyc[0] / steps, cudaGetErrorString(e)); \
  }
  RUNM(0, "stream, per-ks loads")
  RUNM(1, "preloaded, per-ks loads, -Bi per k-step")
  RUNM(6, "preloaded, K-split: all 9 tiles per warp")
  return 0;
}
