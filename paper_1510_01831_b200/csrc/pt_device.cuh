// Device-side data model and PTX helpers shared by the B200 kernels.
//
// Data layout in HBM:
//   * complex128 everywhere as interleaved double2;
//   * Schur inverses S_k^{-1} of a cell: [wz_c][w][w], each block COLUMN-major
//     (element (i,j) at j*w+i) so a CTA streams whole column panels with one
//     1-D bulk copy (cp.async.bulk -> UBLKCP) and thread i reads row i;
//   * Green blocks of a cell: [4 rows r0,r1,rn,rnp][4 slots v0,v1,vn,vnp][w][w], column-major;
//   * outer polarized vectors per RHS: [down(nI,2,wx) | up(nI,2,wx)] exactly like
//     PolarizedTraceStack.flat (sie.py:102-103), RHS-major with a per-RHS stride;
//   * inner vectors identical with (Lc-1, 2, w).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PT_MAX_LC 64
#define PT_THREADS 256

// ---------------------------------------------------------------- geometry

struct LayerInfo {
  int n, off, w, lo, hi;  // interior rows, interior offset, width (= n + 2 npml), kept rows [lo,hi)
  int has_top, has_bot;
  int prow[4];            // layer rows of slot sources v0,v1,vn,vnp: row(1), row(0), row(n+1), row(n)
  double2 coef[4];        // slot coefficients (subdomain.py:157-182)
  long long dense_off;    // double2 offset of the dense inner [pre; pre o op] pair (-1: none)
  long long lu_off;       // double2 offset of the direct inner backend's A^-1 (-1: none)
};

// a[i & 3] without a dynamically indexed (local-memory) array
__device__ __forceinline__ double2 sel4(const double2 (&a)[4], int i) {
  const double2 lo = (i & 1) ? a[1] : a[0], hi = (i & 1) ? a[3] : a[2];
  return (i & 2) ? hi : lo;
}

struct CellInfo {
  int layer, cell, w, wzc, nxc, off, lo, hi;  // cell c of layer: block rows [0,wzc), kept [lo,hi)
  int has_top, has_bot;
  int krow[4];            // block rows of cell slot sources v0,v1,vn,vnp
  int srow[4];            // sampled block rows r0,r1,rn,rnp
  double2 coef[4];        // cell-level slot coefficients
  long long sinv_off;     // double2 offset into the Schur-inverse pool
  long long green_off;    // double2 offset into the Green-block pool
  long long lz_off;       // offset into lz/uz pools
  long long gsmp_off;     // double2 offset into the sampled trace-response pool (-1: none)
  long long q0_off;       // double2 offset into the pass-0 operator pool (-1: none)
};

// Device row layout of a cell's pass-0 operator (pt_problem.q0 rows are (4 w table rows, then (kept row k, output
// row o) k-major); the upload regroups the sample rows by output row so whole 8-row tiles of an output row that no
// job samples are skipped): [4 w Newton-table rows | zero rows up to q0_tab8] then, for o = 0..3 (layer rows 0, 1,
// n, n+1), q0_nk8 rows (o, k) of which the first nk are real.
__host__ __device__ inline int q0_tab8(int w) { return (4 * w + 7) & ~7; }
__host__ __device__ inline int q0_nk8(int nk) { return (nk + 7) & ~7; }
__host__ __device__ inline int q0_rows(int w, int nk) { return q0_tab8(w) + 4 * q0_nk8(nk); }

// A reference to one panel (segment) of a vector: vec < 0 = absent.
struct Ref {
  int vec, seg;
};

// One outer layer-solve job (a boundary_samples / newton_samples / reconstruct call).
struct OJob {
  int layer;
  int vol;           // add the split global source f_l (sie.py:134-151)
  int vfull;         // volume source/output is a full layer slab (no split mask), slab-local rows
  Ref pan[4][2];     // slot panels v0,v1,vn,vnp, each a sum of up to two refs
  int nout;          // sampled layer rows (<=4); -1 = full-volume output (reconstruct)
  int orow[4];       // layer local depths of the sampled rows
  double scoef[4];   // out = scoef*sample + add - (sub0 + sub1)
  Ref dst[4], add[4], sub[4][2];
};

// One inner item: output panel = sum_slot G[cell][row][slot] @ panel_slot + (add0+add1) - (sub0+sub1).
// One inner work item:
//   y   = sum_slot G[cell][row][slot] @ (sgn_slot * (pan[slot][0] + pan[slot][1]))
//   t   = y + (add0 + add1) - (sub0 + sub1)
//   dst = t (mode 0) | rev - t (mode 1) | t - rev (mode 2)
// sgn_slot = -1 when bit slot of flags is set; mode = (flags >> 8) & 3.
struct IItem {
  int cell, row;     // cell < 0: no Green product (pure combination)
  Ref pan[4][2];     // slot panels: pan[s][1] (if present) is added to pan[s][0]
  Ref dst, add[2], sub[2], rev;
  int flags;
  int wgt;           // work weight: number of slot products (1 for a pure combination)
};

// K1 task: one cell, a contiguous range of columns (job, rhs) of its layer.
struct K1Task {
  int cell;          // global cell id (layer-major)
  int jb;            // index into the stage's per-layer job list
  int q0, nq;        // columns [q0, q0+nq) of the layer column space (job-major, R per job)
  long long zoff;    // double2 offset of this task's forward-sweep scratch
};

// ---------------------------------------------------------------- complex helpers

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc += a*b
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// conj(a)*b
__device__ __forceinline__ double2 cconjmul(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

// coherent (L2) load for data produced earlier in the same kernel by other CTAs/threads
__device__ __forceinline__ double2 ld_cg(const double2* p) { return __ldcg(p); }

// ---------------------------------------------------------------- mbarrier + bulk copy (TMA)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// expect_tx without release semantics: the producer thread does not wait for its earlier memory operations
// (the bulk copies it has in flight) before arming the barrier
__device__ __forceinline__ void mbar_expect_tx_relaxed(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// wait with a suspend-time hint: the thread sleeps in the barrier unit until the phase completes
// (or the hint expires), so a waiting producer lane does not steal issue slots from its SMSP
__device__ __forceinline__ void mbar_wait_suspend(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// wait with exponential nanosleep backoff: for a lone producer thread whose spinning would
// otherwise steal issue slots from the consumer warps of its SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ns = 32;
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : 256;
  }
}
// 1-D bulk async copy global -> shared, completion counted on an mbarrier (SASS UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// multicast variant: the same bytes land at the same smem offset of every CTA in ctaMask,
// each CTA's mbarrier at the same offset receives the complete_tx
__device__ __forceinline__ void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Relaxed arrive: no release fence.  For consumers releasing a ring slot whose shared-memory
// contents have already been consumed by executed instructions: a release arrive would wait for
// ALL outstanding memory operations of the thread (prefetch loads a step ahead, global stores),
// serialising every chunk on HBM latency.
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// shared::cta address of this CTA -> the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 16-byte DSMEM store that counts its bytes on the destination CTA's mbarrier
__device__ __forceinline__ void st_async_c(uint32_t cluster_addr, double2 v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                   cluster_addr),
               "d"(v.x), "d"(v.y), "r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// FP64 tensor-core MMA: C(8x8) += A(8x4) B(4x8), one double of A, B and two of C per thread
// (row-major A fragment: row = lane/4, k = lane%4; col-major B: k = lane%4, col = lane/4;
//  C: row = lane/4, cols 2*(lane%4) and +1).  SASS: DMMA.8x8x4.
__device__ __forceinline__ void dmma_f64(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 16-byte global -> shared async copy (LDGSTS), L2 only (.cg: coherent with data written by other
// CTAs before a cluster barrier); pred = false zero-fills the destination
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(pred ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------- reductions

// block-wide sum of one double (all threads get the result); red: >= 32 doubles of smem
// two block sums with one pair of barriers (red: >= 2 * warps doubles); fixed order: deterministic
__device__ __forceinline__ double2 block_sum2(double a, double b, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    red[2 * wid] = a;
    red[2 * wid + 1] = b;
  }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
  const int nw = (blockDim.x + 31) >> 5;
  for (int i = 0; i < nw; ++i) {
    sa += red[2 * i];
    sb += red[2 * i + 1];
  }
  return make_double2(sa, sb);
}
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  const int nw = (blockDim.x + 31) >> 5;
  for (int i = 0; i < nw; ++i) s += red[i];  // fixed order: deterministic
  return s;
}
