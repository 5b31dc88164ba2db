// K1: batched cell solves H_c X = B with a TWISTED block-tridiagonal
// factorization (replaces SuperLU.solve, subdomain.py:214-221).
//
// With m = wz_c/2 the offline stage stores S_k^{-1} (k < m, top Schur
// complements), T_k^{-1} (k > m, bottom Schur complements) and M^{-1} (k = m),
// see offline._twisted_inverses.  A solve is two half-length chains that run
// concurrently on a CTA pair of one thread-block cluster:
//
//   top    z_k = S_k^{-1}(b_k - l_k z_{k-1}),  k = 0..m-1
//   bottom y_k = T_k^{-1}(b_k - u_k y_{k+1}),  k = wz_c-1..m+1
//   middle x_m = M^{-1}(b_m - l_m z_{m-1} - u_m y_{m+1})   (vectors swapped over DSMEM)
//   top    x_k = z_k - u_k S_k^{-1} x_{k+1},   k = m-1..0
//   bottom x_k = y_k - l_k T_k^{-1} x_{k-1},   k = m+1..wz_c-1
//
// so the dependent chain is wz_c+1 block matvecs instead of 2 wz_c - 1.
// A cluster is 2*CM CTAs: CM column CTAs per half, each owning NC right-hand
// side columns (a column = one (layer-solve job, RHS) pair).  The factor
// blocks do not depend on data: a producer warp streams them through an
// NS-slot shared-memory ring with 1-D bulk async copies (cp.async.bulk ->
// SASS UBLKCP), multicast to the CM CTAs of the half that consume the same
// block; consumers release slots through mbarriers, so no CTA-wide barrier
// guards the ring.
//
// The right-hand side b_k is generated in the prologue of every step from the
// job description (equivalent interface sources at the four cut rows, the
// split volume source, the cell trace sources on the reconstruction pass), so
// no layer volume is ever materialised; the epilogue writes only what the
// caller consumes (four Newton rows per cell, the sampled layer rows, or the
// stitched volume).
#include <cooperative_groups.h>

#include <algorithm>

#include "pt_launch.cuh"

namespace cg = cooperative_groups;

struct ColInfo {
  int jid, r, panmask, vol, nout, vfull, opos[4], pad[6];
};

template <int NC>
__global__ void __launch_bounds__(K1_THREADS, 1) k1_twisted(const K1Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int CM = p.cm;
  const int h = rank / CM, cm = rank - h * CM;
  const K1Task task = p.tasks[blockIdx.x / (2 * CM)];
  const CellInfo cell = p.cells[task.cell];
  const LayerInfo lay = p.layers[cell.layer];
  const int w = cell.w, wzc = cell.wzc;
  const int m = wzc >> 1, mb = wzc - 1 - m;
  const int nst = h == 0 ? 2 * m + 1 : 2 * mb + 1;
  const int tid = threadIdx.x;
  constexpr int NS = K1_NS;  // power of two: slot = c & (NS-1), use = c >> log2(NS)
  const int nIc = p.Lc - 1;

  unsigned char* ring = smem;
  double2* VA = reinterpret_cast<double2*>(ring + (size_t)NS * p.slot_bytes);
  double2* VB = VA + w * NC;
  double2* XC = VB + w * NC;  // partner's half-chain vector at the middle block
  double2* red = XC + w * NC;
  ColInfo* cols = reinterpret_cast<ColInfo*>(red + K1_CONSUMERS * NC);
  uint64_t* full = reinterpret_cast<uint64_t*>(cols + NC);
  uint64_t* lempty = full + NS;
  uint64_t* cempty = lempty + NS;
  uint64_t* xbar = cempty + NS;

  const int jc = max(1, min(w, p.slot_bytes / (w * 16)));
  const int nch = (w + jc - 1) / jc;
  const int total = nst * nch;
  const double2* S = p.sinv + cell.sinv_off;
  // factor block used by step s of this half
  auto kblk = [&](int s) -> int {
    if (h == 0) return s <= m ? s : 2 * m - s;
    return s < mb ? wzc - 1 - s : (s == mb ? m : m + (s - mb));
  };

  if (tid < NC) {
    ColInfo ci;
    ci.jid = -1;
    ci.r = 0;
    ci.panmask = ci.vol = ci.nout = ci.vfull = 0;
    const int ql = cm * NC + tid;
    if (ql < task.nq) {
      const int q = task.q0 + ql;
      if (p.pass == 2) {
        ci.jid = 0;
        ci.r = q;
      } else {
        ci.jid = p.ljobs[task.jb + q / p.R];
        ci.r = q % p.R;
        const OJob& jb = p.jobs[ci.jid];
        int msk = 0;
        for (int s = 0; s < 4; ++s)
          if (jb.pan[s][0].vec >= 0) msk |= 1 << s;
        ci.panmask = msk;
        ci.vol = jb.vol ? (jb.vfull ? 2 : 1) : 0;
        ci.vfull = jb.vfull;
        ci.nout = jb.nout;
        for (int o = 0; o < 4; ++o) ci.opos[o] = o < jb.nout ? jb.orow[o] + p.npml - 1 : -1;
      }
    }
    cols[tid] = ci;
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&lempty[s], K1_CONSUMERS / 32);
      mbar_init(&cempty[s], CM);
    }
    mbar_init(xbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  cl.sync();  // every barrier of the cluster is initialised before any remote traffic
  if (tid == 0) mbar_expect_tx(xbar, (uint32_t)(w * NC * 16));

  if (tid >= K1_CONSUMERS) {
    // ------------------------------------------------------------ producer warp
    if (tid == K1_CONSUMERS) {
      const uint16_t mask = (uint16_t)(((1u << CM) - 1u) << (h * CM));
      for (int c = 0; c < total; ++c) {
        const int slot = c & (NS - 1), u = c >> K1_NS_LOG2;
        if (u > 0) mbar_wait(&lempty[slot], (uint32_t)((u - 1) & 1));
        const int s = c / nch, ch = c - s * nch;
        const int c0 = ch * jc, cw = min(jc, w - c0);
        const uint32_t bytes = (uint32_t)cw * w * 16u;
        mbar_expect_tx(&full[slot], bytes);
        const int issuer = slot % CM;
        const double2* src = S + (size_t)kblk(s) * w * w + (size_t)c0 * w;
        unsigned char* dst = ring + (size_t)slot * p.slot_bytes;
        if (CM == 1) {
          bulk_g2s(dst, src, bytes, &full[slot]);
        } else {
          if (u > 0) mbar_arrive_remote(mapa(&cempty[slot], (uint32_t)(h * CM + issuer)));
          if (issuer == cm) {
            if (u > 0) mbar_wait(&cempty[slot], (uint32_t)((u - 1) & 1));
            bulk_g2s_mc(dst, src, bytes, &full[slot], mask);
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const int G = K1_CONSUMERS / w;
    const bool mact = tid < G * w;
    const int mi = tid % w, mg = tid / w;
    double2* Z = p.Z + task.zoff + (size_t)cm * wzc * w * NC;

    auto rhs = [&](int k, int j, int q) -> double2 {
      const ColInfo& ci = cols[q];
      if (ci.jid < 0) return czero();
      if (p.pass == 2) return p.bd[((size_t)ci.r * wzc + k) * w + j];
      double2 inner = czero();
      if (k >= cell.lo && k < cell.hi) {
        const int X = cell.off + k;
#pragma unroll
        for (int sl = 0; sl < 4; ++sl)
          if ((ci.panmask >> sl & 1) && j == lay.prow[sl])
            inner = cadd(inner, cmul(lay.coef[sl], p.P[((size_t)(ci.jid * 4 + sl) * p.R + ci.r) * p.wx + X]));
        if (ci.vol == 1 && j >= lay.lo && j < lay.hi)
          inner = cadd(inner, p.f[ci.r * p.f_stride + (size_t)(lay.off + j) * p.wx + X]);
        else if (ci.vol == 2)
          inner = cadd(inner, p.f[ci.r * p.f_stride + (size_t)j * p.wx + X]);
      }
      if (p.pass == 1) {
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {
          const bool has = sl < 2 ? cell.has_top : cell.has_bot;
          if (has && k == cell.krow[sl]) {
            const int I = sl < 2 ? cell.cell - 1 : cell.cell;
            const double2 t = p.tr[((((size_t)ci.jid * p.R + ci.r) * nIc + I) * 2 + (sl & 1)) * p.wmax + j];
            return cadd(cmul(cell.coef[sl], t), inner);
          }
        }
      }
      return inner;
    };

    auto emit = [&](int k, int e, double2 x) {
      const int i = e / NC, q = e - (e / NC) * NC;
      const ColInfo& ci = cols[q];
      if (ci.jid < 0) return;
      if (p.pass == 2) {
        p.xd[((size_t)ci.r * wzc + k) * w + i] = x;
      } else if (p.pass == 0) {
#pragma unroll
        for (int idx = 0; idx < 4; ++idx) {
          const bool need = idx < 2 ? cell.has_top : cell.has_bot;
          if (need && k == cell.srow[idx])
            p.tables[((((size_t)ci.jid * p.Lc + cell.cell) * 4 + idx) * p.R + ci.r) * p.wmax + i] = x;
        }
      } else if (k >= cell.lo && k < cell.hi) {
        const int X = cell.off + k;
        if (ci.nout < 0) {
          if (ci.vfull)
            p.u[ci.r * p.u_stride + (size_t)i * p.wx + X] = x;
          else if (i >= lay.lo && i < lay.hi)
            p.u[ci.r * p.u_stride + (size_t)(lay.off + i) * p.wx + X] = x;
        } else {
#pragma unroll
          for (int o = 0; o < 4; ++o)
            if (i == ci.opos[o]) p.smp[((size_t)(ci.jid * 4 + o) * p.R + ci.r) * p.wx + X] = x;
        }
      }
    };

    const int nel = w * NC;
    double2* cur = VA;
    double2* nxt = VB;
    int c = 0;
    const int partner = (1 - h) * CM + cm;
    auto kind_of = [&](int s) -> int {
      return (h == 0) ? (s < m ? 0 : (s == m ? 1 : 2)) : (s < mb ? 0 : (s == mb ? 1 : 2));
    };
    // per-thread operand of a step that does not depend on the chain: b_k (elimination and
    // middle steps) or the stored z_k / y_k (back-substitution).  Loaded one step ahead so the
    // global-load latency overlaps the previous step's matvec.
    auto pre_load = [&](int s, double2* v) {
      const int kb = kblk(s);
      const int kd = kind_of(s);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int e = tid + t * K1_CONSUMERS;
        if (e < nel) v[t] = kd == 2 ? Z[(size_t)kb * nel + e] : rhs(kb, e / NC, e - (e / NC) * NC);
      }
    };
    double2 pv[4];
    pre_load(0, pv);
    for (int s = 0; s < nst; ++s) {
      const int kb = kblk(s);
      const int kind = kind_of(s);
      double2 zr[4];
      // ---- prologue: matvec input in cur (in place: every thread owns the same elements throughout)
      if (kind == 0) {
        const double2 cf = h == 0 ? p.lz[cell.lz_off + kb] : p.uz[cell.lz_off + kb];
        const bool first = s == 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int e = tid + t * K1_CONSUMERS;
          if (e < nel) cur[e] = first ? pv[t] : csub(pv[t], cmul(cf, cur[e]));
        }
      } else if (kind == 1) {
        const uint32_t rx = mapa(XC, (uint32_t)partner), rb = mapa(xbar, (uint32_t)partner);
        for (int e = tid; e < nel; e += K1_CONSUMERS) st_async_c(rx + (uint32_t)e * 16u, cur[e], rb);
        mbar_wait(xbar, 0);
        const double2 lm = p.lz[cell.lz_off + m], um = p.uz[cell.lz_off + m];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int e = tid + t * K1_CONSUMERS;
          if (e < nel) {
            const double2 zt = h == 0 ? cur[e] : XC[e];  // z_{m-1} (top chain)
            const double2 yb = h == 0 ? XC[e] : cur[e];  // y_{m+1} (bottom chain)
            cur[e] = csub(csub(pv[t], cmul(lm, zt)), cmul(um, yb));
          }
        }
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) zr[t] = pv[t];
      }
      if (s + 1 < nst) pre_load(s + 1, pv);
      named_bar(1, K1_CONSUMERS);
      // ---- y = Blk[kb] cur
      double2 acc[NC], acc2[NC];
#pragma unroll
      for (int q = 0; q < NC; ++q) acc[q] = acc2[q] = czero();
      for (int ch = 0; ch < nch; ++ch, ++c) {
        const int slot = c & (NS - 1);
        mbar_wait(&full[slot], (uint32_t)((c >> K1_NS_LOG2) & 1));
        const double2* blk = reinterpret_cast<const double2*>(ring + (size_t)slot * p.slot_bytes);
        const int c0 = ch * jc, cw = min(jc, w - c0);
        if (mact) {
          int jj = mg;
          for (; jj + G < cw; jj += 2 * G) {
            const double2 a0 = blk[jj * w + mi], a1 = blk[(jj + G) * w + mi];
            const double2* t0 = cur + (c0 + jj) * NC;
            const double2* t1 = cur + (c0 + jj + G) * NC;
#pragma unroll
            for (int q = 0; q < NC; ++q) {
              cfma(acc[q], a0, t0[q]);
              cfma(acc2[q], a1, t1[q]);
            }
          }
          if (jj < cw) {
            const double2 a0 = blk[jj * w + mi];
            const double2* t0 = cur + (c0 + jj) * NC;
#pragma unroll
            for (int q = 0; q < NC; ++q) cfma(acc[q], a0, t0[q]);
          }
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&lempty[slot]);
      }
      if (mact) {
#pragma unroll
        for (int q = 0; q < NC; ++q) red[(mg * w + mi) * NC + q] = cadd(acc[q], acc2[q]);
      }
      named_bar(1, K1_CONSUMERS);
      // ---- epilogue
      const double2 cf = kind == 2 ? (h == 0 ? p.uz[cell.lz_off + kb] : p.lz[cell.lz_off + kb]) : czero();
      for (int t = 0; t < 4; ++t) {
        const int e = tid + t * K1_CONSUMERS;
        if (e >= nel) break;
        const int i = e / NC, q = e - (e / NC) * NC;
        double2 y = red[i * NC + q];
        for (int g = 1; g < G; ++g) y = cadd(y, red[(g * w + i) * NC + q]);
        if (kind == 0) {
          nxt[e] = y;
          Z[(size_t)kb * nel + e] = y;
        } else if (kind == 1) {
          nxt[e] = y;
          if (h == 0) emit(m, e, y);
        } else {
          const double2 x = csub(zr[t], cmul(cf, y));
          nxt[e] = x;
          emit(kb, e, x);
        }
      }
      double2* tmp = cur;
      cur = nxt;
      nxt = tmp;
    }
  }
  __syncwarp();
  cl.sync();  // no CTA leaves while a partner may still write into its shared memory
}

size_t k1_smem_bytes(int wmax, int nc, int slot_bytes, int ns) {
  (void)ns;
  ns = K1_NS;
  return (size_t)ns * slot_bytes + (size_t)(3 * wmax + K1_CONSUMERS) * nc * 16 + (size_t)nc * sizeof(ColInfo) +
         (size_t)(3 * ns + 1) * 8 + 128;
}

cudaError_t k1_launch(const K1Params& p0, int ntasks, int nc, int wmax, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  if (nc * wmax > 4 * K1_CONSUMERS) return cudaErrorInvalidValue;  // epilogue holds <= 4 elements/thread
  static int maxsm = 0;
  if (!maxsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  // ring slots as large as the shared memory left next to this NC's vectors allows (<= 48 KB)
  K1Params p = p0;
  const long long fixed = (long long)k1_smem_bytes(wmax, nc, 0, K1_NS);
  long long slot = std::min(((long long)maxsm - fixed) / K1_NS, 49152LL) / 16 * 16;
  if (slot < 16LL * wmax) return cudaErrorInvalidValue;
  p.slot_bytes = (int)slot;
  p.ns = K1_NS;
  const size_t smax = k1_smem_bytes(wmax, nc, p.slot_bytes, K1_NS);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ntasks * 2 * p.cm, 1, 1);
  cfg.blockDim = dim3(K1_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smax;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * p.cm;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (nc) {
#define PT_K1_CASE(N)                                                                                 \
  case N:                                                                                             \
    cudaFuncSetAttribute(k1_twisted<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);     \
    if (2 * p.cm > 8) cudaFuncSetAttribute(k1_twisted<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); \
    return cudaLaunchKernelEx(&cfg, k1_twisted<N>, p);
    PT_K1_CASE(1)
    PT_K1_CASE(2)
    PT_K1_CASE(4)
    PT_K1_CASE(8)
#undef PT_K1_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
