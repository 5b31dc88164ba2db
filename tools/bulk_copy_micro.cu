// Per-SM throughput of 1-D bulk copies (cp.async.bulk, UBLKCP) vs cp.async (LDGSTS) for small pieces,
// L2-resident source: one CTA per SM copies NB pieces of SZ bytes into shared memory and waits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1510_01831_b200/csrc -o tools/bulk_copy_micro tools/bulk_copy_micro.cu
#include <cstdio>
#include "pt_device.cuh"

__global__ void k_bulk(const double2* src, int nb, int sz, int reps, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const char* s = reinterpret_cast<const char*>(src) + (size_t)blockIdx.x * 256 * 1024;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar, (uint32_t)(nb * sz));
      for (int i = 0; i < nb; ++i) bulk_g2s(sm + (size_t)i * sz, s + (size_t)i * sz, sz, &bar);
    }
    mbar_wait(&bar, r & 1);
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

__global__ void k_ldgsts(const double2* src, int nb, int sz, int reps, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const char* s = reinterpret_cast<const char*>(src) + (size_t)blockIdx.x * 256 * 1024;
  long long t0 = clock64();
  const int tot = nb * sz / 16;
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < tot; i += blockDim.x) cp_async16(sm + (size_t)i * 16, s + (size_t)i * 16, true);
    cp_async_wait_all();
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  double2* src;
  cudaMalloc(&src, 148ull * 256 * 1024 + 1024 * 1024);
  cudaMemset(src, 0, 148ull * 256 * 1024);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  const int reps = 200;
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int sz : {1024, 2048, 4096, 16384}) {
    for (int nb : {1, 4, 16, 48}) {
      if (nb * sz > 196 * 1024) continue;
      k_bulk<<<148, 256, 200 * 1024>>>(src, nb, sz, reps, d);
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      const double cb = (double)h[0] / reps;
      k_ldgsts<<<148, 256, 200 * 1024>>>(src, nb, sz, reps, d);
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      const double cl = (double)h[0] / reps;
      printf("piece %6d B x %3d: bulk %7.0f cyc (%.1f B/cyc)   ldgsts %7.0f cyc (%.1f B/cyc)  %s\n", sz, nb, cb,
             nb * sz / cb, cl, nb * sz / cl, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
