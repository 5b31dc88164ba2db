// Grid-barrier cost on the B200: cooperative-groups grid.sync() vs a sense-reversing barrier on one global
// counter (red.release + ld.acquire spin), 148 CTAs x 256 threads (one per SM), 1000 barriers each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridsync_micro tools/gridsync_micro.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

__device__ unsigned int g_count = 0, g_gen = 0;
__device__ __forceinline__ void bar_custom(unsigned nblk, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned my = gen + 1;
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(&g_count) : "memory");
    if (old == nblk * my - 1) {
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&g_gen), "r"(my) : "memory");
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_gen) : "memory");
      } while (v < my);
    }
    gen = my;
  }
  __syncthreads();
}
__global__ void k_custom(int iters, unsigned long long* out) {
  unsigned gen = 0;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) bar_custom(gridDim.x, gen);
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  unsigned long long h[1024];
  int iters = 1000;
  for (int smem : {0, 200 * 1024}) {
    cudaFuncSetAttribute(k_cg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_custom, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    void* args[] = {&iters, &d};
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, nsm, 256, args, smem, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
      printf("cg grid.sync   smem %6d: %.3f us per barrier (events), cta0 %.0f cycles per barrier  err=%s\n", smem,
             ms * 1e3 / iters, (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_custom, nsm, 256, args, smem, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
      printf("custom barrier smem %6d: %.3f us per barrier (events), cta0 %.0f cycles per barrier  err=%s\n", smem,
             ms * 1e3 / iters, (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
      unsigned z = 0;
      cudaMemcpyToSymbol(g_count, &z, 4);
      cudaMemcpyToSymbol(g_gen, &z, 4);
    }
  }
  return 0;
}
