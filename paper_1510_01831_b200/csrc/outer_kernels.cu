// Outer-level kernels: equivalent-source panel gather, sample combination,
// polarized-vector algebra, fused MGS Arnoldi, and the true residual (K5).
//
// Outer vectors are RHS-major: element e of RHS r of view V lives at
// V.p[r * V.stride + e]; panels (segments) are wx long.  Stage kernels run on
// the compacted list of still-active RHS (rmap), so converged right-hand sides
// cost nothing and never feed garbage into an inner solve.
#include <cooperative_groups.h>

#include "pt_device.cuh"

#include <algorithm>

#include <cstdlib>
#include "pt_launch.cuh"
#include "stage_dev.cuh"




__global__ void k_gather_panels(const OJob* jobs, int njobs, VecTab t, const int* rmap, int nq, int wx,
                                double2* P) {
  const long long total = (long long)njobs * 4 * nq * wx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    gather_elem(jobs, t, rmap, nq, wx, P, e);
}

__global__ void k_combine(const OJob* jobs, int njobs, VecTab t, const int* rmap, int nq, int wx,
                          const double2* smp) {
  const long long total = (long long)njobs * 4 * nq * wx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    combine_elem(jobs, t, rmap, nq, wx, smp, e);
}

template <bool DIRECT, bool SEG>
__global__ void __launch_bounds__(P0_KQ * 32) k_pass0(const int* __restrict__ grp, const int* __restrict__ ljobs,
                                                      const OJob* __restrict__ jobs,
                                                      const CellInfo* __restrict__ cells,
                                                      const LayerInfo* __restrict__ layers,
                                                      const double2* __restrict__ q0, const double2* __restrict__ P,
                                                      double2* __restrict__ tables, double2* __restrict__ smp, int R,
                                                      int Lc, int wx, int wmax, int accum, VecTab tab,
                                                      const int* rmap, int direct, RhsOut ro) {
  __shared__ double part[(P0_KQ - 1) * 2 * 4 * 32];
  pass0_item<DIRECT, SEG>(grp, ljobs, jobs, cells, layers, q0, P, tables, smp, R, Lc, wx, wmax, blockIdx.x / Lc,
                     blockIdx.x % Lc, blockIdx.y, blockIdx.z, threadIdx.x >> 5, part, 1, accum,
                     DIRECT ? &tab : nullptr, rmap, ro.base ? &ro : nullptr);
}

__global__ void __launch_bounds__(GS_WARPS * 32) k_green_samples(
    const OJob* __restrict__ jobs, const CellInfo* __restrict__ cells, const LayerInfo* __restrict__ layers,
    const double2* __restrict__ gsmp, const double2* __restrict__ tr, double2* __restrict__ smp, int R, int Lc, int wx,
    int wmax, VecTab tab, const int* rmap, int fuse_combine) {
  extern __shared__ double2 trs[];  // [4 slots][w4][8 rhs]
  green_item(jobs, cells, layers, gsmp, tr, smp, R, Lc, wx, wmax, blockIdx.x, blockIdx.y, blockIdx.z, trs,
             fuse_combine ? &tab : nullptr, rmap);
}

// Sampled trace response, many-warp form: CTA = (job x cell, GS2_NG groups of 8 RHS, GS2_TPC row tiles);
// each row tile's K = (slot, column) range is split over GS2_KQ warps (A loads of a warp issued 8 k-steps
// at a time), every A fragment serves all GS2_NG RHS groups, and the partial tiles are summed in a fixed
// order by the kq = 0 warp.  Same products as green_item; the sum over K is split in GS2_KQ parts.
// KQ = 1, TPC = 8 (one warp per row tile over the whole K, eight row tiles per CTA): the staged trace panels
// serve 8 row tiles instead of 2 (cfg5 64 RHS: 263 -> 157 us per sweep-stage launch; KQ 4 / TPC 2 was tuned on
// cfg2's 16 RHS in round 1)
#ifndef GS2_KQ
#define GS2_KQ 1
#endif
#ifndef GS2_TPC
#define GS2_TPC 8
#endif
#ifndef GS2_NG
#define GS2_NG 2
#endif
__global__ void __launch_bounds__(GS2_KQ * GS2_TPC * 32) k_green_samples2(
    const OJob* __restrict__ jobs, const CellInfo* __restrict__ cells, const LayerInfo* __restrict__ layers,
    const double2* __restrict__ gsmp, const double2* __restrict__ tr, double2* __restrict__ smp, int R, int Lc, int wx,
    int wmax, VecTab tab, const int* rmap, int fuse_combine) {
  extern __shared__ double2 trs[];  // [4 slots][w4][8 GS2_NG rhs], then the partial tiles
  const int jid = blockIdx.x / Lc, c = blockIdx.x - jid * Lc;
  const OJob& jb = jobs[jid];
  const int nout = jb.nout;
  if (nout <= 0) return;
  const LayerInfo& lay = layers[jb.layer];
  const CellInfo& ci = cells[jb.layer * Lc + c];
  const int w = ci.w, w4 = (w + 3) & ~3, nIc = Lc - 1, tid = threadIdx.x;
  const int lane = tid & 31, wp = tid >> 5;
  const int nrows = (ci.hi - ci.lo) * nout;  // (k, o) rows of this cell, k-major
  if (blockIdx.z * GS2_TPC * 8 >= nrows) return;  // whole CTA: no barrier is skipped by part of it
  constexpr int NR = 8 * GS2_NG;
  const int r0 = blockIdx.y * NR, nr = min(NR, R - r0);
  const int s_lo = ci.has_top ? 0 : 2, s_hi = ci.has_bot ? 4 : 2;
  {
    // trace panels of the used slots -> trs[sl][j][rr]: 8 independent loads in flight per thread, then the
    // stores (a load-store loop would serialise one L2 round trip per element)
    const int ne = (s_hi - s_lo) * NR * w4;
    for (int e0 = tid; e0 < ne; e0 += 8 * GS2_KQ * GS2_TPC * 32) {
      double2 v[8];
      int dsti[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * GS2_KQ * GS2_TPC * 32;
        v[u] = make_double2(0.0, 0.0);
        dsti[u] = -1;
        if (e < ne) {
          const int j = e % w4, rest = e / w4, rr = rest % NR, sl = s_lo + rest / NR;
          const int I = sl < 2 ? c - 1 : c;
          const bool okr = rr < nr && I >= 0 && I < nIc && j < w;
          if (okr) v[u] = __ldg(tr + (((size_t)(jid * R + r0 + rr) * nIc + I) * 2 + (sl & 1)) * wmax + j);
          dsti[u] = (sl * w4 + j) * NR + rr;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (dsti[u] >= 0) trs[dsti[u]] = v[u];
    }
  }
  __syncthreads();
  const int t = wp / GS2_KQ, kq = wp - t * GS2_KQ;
  const int tile = blockIdx.z * GS2_TPC + t;
  const int ar = lane >> 2, ak = lane & 3;
  const int m = tile * 8 + ar;
  const bool mok = m < nrows;
  const int mk = mok ? m / nout : 0, mo = mok ? m - (m / nout) * nout : 0;
  const int orow = jb.orow[mo];
  const int oi = orow == 0 ? 0 : (orow == 1 ? 1 : (orow == lay.n ? 2 : 3));
  const double2* grow = gsmp + ci.gsmp_off + ((size_t)(ci.lo + mk) * 4 + oi) * 4 * w;  // [4 slots][w]
  const int kps = w4 >> 2, nks = (s_hi - s_lo) * kps;
  const int kb = kq * nks / GS2_KQ, ke = (kq + 1) * nks / GS2_KQ;
  double acc[GS2_NG][4];
#pragma unroll
  for (int g = 0; g < GS2_NG; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.0;
  if (tile * 8 < nrows) {
    // (slot, k-step within the slot) advanced incrementally (no divisions in the unrolled loops)
    int sl_c = s_lo + kb / kps, r_c = kb - (kb / kps) * kps;
    for (int ks0 = kb; ks0 < ke; ks0 += 8) {
      double2 av[8];
      int sls[8], js[8];
      {
        int sl = sl_c, r = r_c;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          sls[u] = sl;
          js[u] = r * 4 + ak;
          if (++r == kps) {
            r = 0;
            ++sl;
          }
        }
        sl_c = sl;
        r_c = r;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int sl = sls[u], j = js[u];
        av[u] = (ks0 + u < ke && mok && j < w) ? __ldg(grow + sl * w + j) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int ks = ks0 + u;
        if (ks >= ke) break;
        const int sl = sls[u], j = js[u];
        const double2* tb = trs + ((size_t)sl * w4 + j) * NR + ar;
#pragma unroll
        for (int g = 0; g < GS2_NG; ++g) {
          const double2 bv = tb[g * 8];
          dmma_f64(acc[g][0], acc[g][1], av[u].x, bv.x);
          dmma_f64(acc[g][2], acc[g][3], av[u].x, bv.y);
          dmma_f64(acc[g][0], acc[g][1], -av[u].y, bv.y);
          dmma_f64(acc[g][2], acc[g][3], av[u].y, bv.x);
        }
      }
    }
  }
  double* part = reinterpret_cast<double*>(trs + (size_t)4 * w4 * NR);  // [TPC][KQ-1][NG][4][32]
  if (kq > 0) {
#pragma unroll
    for (int g = 0; g < GS2_NG; ++g)
#pragma unroll
      for (int q = 0; q < 4; ++q) part[((((size_t)t * (GS2_KQ - 1) + kq - 1) * GS2_NG + g) * 4 + q) * 32 + lane] = acc[g][q];
  }
  __syncthreads();
  if (kq > 0 || !mok) return;
#pragma unroll
  for (int p2 = 0; p2 < GS2_KQ - 1; ++p2)
#pragma unroll
    for (int g = 0; g < GS2_NG; ++g)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[g][q] += part[((((size_t)t * (GS2_KQ - 1) + p2) * GS2_NG + g) * 4 + q) * 32 + lane];
  // C fragment: row ar, columns (RHS) 2 ak and 2 ak + 1 of each group
#pragma unroll
  for (int g = 0; g < GS2_NG; ++g)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rr = g * 8 + 2 * ak + h;
      if (rr >= nr) continue;
      double2* dst = smp + ((size_t)(jid * 4 + mo) * R + r0 + rr) * wx + ci.off + ci.lo + mk;
      const double2 yv = cadd(*dst, h == 0 ? make_double2(acc[g][0], acc[g][2]) : make_double2(acc[g][1], acc[g][3]));
      if (!fuse_combine) {
        *dst = yv;
      } else {  // combine fused in: out = scoef*sample + add - (sub0 + sub1) (k_combine)
        const int xg = ci.off + ci.lo + mk, r = rmap[r0 + rr];
        double2 o = cscale(yv, jb.scoef[mo]);
        if (jb.add[mo].vec >= 0) o = cadd(o, vref(tab, jb.add[mo], r, xg, wx));
        if (jb.sub[mo][0].vec >= 0) {
          double2 sb = vref(tab, jb.sub[mo][0], r, xg, wx);
          if (jb.sub[mo][1].vec >= 0) sb = cadd(sb, vref(tab, jb.sub[mo][1], r, xg, wx));
          o = csub(o, sb);
        }
        const VecView& dv = tab.v[jb.dst[mo].vec];
        dv.p[(size_t)r * dv.stride + (size_t)jb.dst[mo].seg * wx + xg] = o;
      }
    }
}

// Direct inner backend (nested.py:156-254, backend="lu"): traces x = A^-1 b per (job, RHS), A^-1 the layer's
// inverted cell-interface system (m = 2 nI w, row-major), b_i = (Newton row n of cell i, row 1 of cell i+1)
// from the tables, x_i -> traces (nI, 2, w).  CTA = (8-row tile, job, 16 RHS); P0_KQ warps split K, partial
// tiles summed in a fixed order; DMMA m8n8k4 f64, complex as 4 real products.  Accounting as the reference's
// substitutions: 4 w^2 (4 nI - 3) touches per instance (TouchCounter, nested.py:67-73).
__global__ void __launch_bounds__(P0_KQ * 32) k_inner_lu(const int* __restrict__ stage_jobs, const OJob* __restrict__ jobs,
                                                       const LayerInfo* __restrict__ layers,
                                                       const double2* __restrict__ lu,
                                                       const double2* __restrict__ tables, double2* __restrict__ trc,
                                                       int R, int Lc, int wmax, unsigned long long* counters) {
  __shared__ double part[(P0_KQ - 1) * 2 * 4 * 32];
  const int job = stage_jobs[blockIdx.y];
  const LayerInfo& lay = layers[jobs[job].layer];
  const int w = lay.w, nI = Lc - 1, m = 2 * nI * w;
  const int tile = blockIdx.x, n0 = blockIdx.z * 16;
  if (tile * 8 >= m || n0 >= R) return;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int ar = lane >> 2, ak = lane & 3;
  const double2* arow = lu + lay.lu_off + (size_t)min(tile * 8 + ar, m - 1) * m + ak;
  const bool aok = tile * 8 + ar < m;
  // b[k] for RHS column q: k = (i, h, j) -> tables[job][cell i + h][h ? r1 : rn][q][j]
  auto bval = [&](int k, int q) -> double2 {
    const int i = k / (2 * w), rem = k - i * 2 * w, h = rem / w, j = rem - h * w;
    return __ldg(tables + ((((size_t)job * Lc + i + h) * 4 + (h ? 1 : 2)) * R + q) * wmax + j);
  };
  double acc[2][4];
#pragma unroll
  for (int g = 0; g < 2; ++g) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.0;
  const int nks = (m + 3) >> 2;
  const int kb = wp * nks / P0_KQ, ke = (wp + 1) * nks / P0_KQ;
  for (int ks0 = kb; ks0 < ke; ks0 += 8) {
    double2 av[8], bv[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = (ks0 + u) * 4 + ak;
      const bool kin = ks0 + u < ke && k < m;
      av[u] = kin && aok ? __ldg(arow + (size_t)(ks0 + u) * 4) : make_double2(0.0, 0.0);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int q = n0 + g * 8 + ar;
        bv[u][g] = kin && q < R ? bval(k, q) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        dmma_f64(acc[g][0], acc[g][1], av[u].x, bv[u][g].x);
        dmma_f64(acc[g][2], acc[g][3], av[u].x, bv[u][g].y);
        dmma_f64(acc[g][0], acc[g][1], -av[u].y, bv[u][g].y);
        dmma_f64(acc[g][2], acc[g][3], av[u].y, bv[u][g].x);
      }
  }
  if (wp > 0)
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int t = 0; t < 4; ++t) part[(((wp - 1) * 2 + g) * 4 + t) * 32 + lane] = acc[g][t];
  __syncthreads();
  if (wp > 0) return;
#pragma unroll
  for (int p2 = 0; p2 < P0_KQ - 1; ++p2)
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[g][t] += part[((p2 * 2 + g) * 4 + t) * 32 + lane];
  const int row = tile * 8 + ar;
  if (row < m) {
    const int i = row / (2 * w), rem = row - i * 2 * w, h = rem / w, j = rem - h * w;
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int q = n0 + g * 8 + 2 * ak + hh;
        if (q < R)
          trc[(((size_t)job * R + q) * nI + i) * 2 * wmax + (size_t)h * wmax + j] =
              make_double2(acc[g][hh], acc[g][2 + hh]);
      }
  }
  if (tile == 0 && threadIdx.x == 0) {
    const int nq = min(16, R - n0);
    atomicAdd(&counters[1], (unsigned long long)nq * 4ULL * w * w * (4ULL * nI - 3ULL));
    atomicAdd(&counters[2], (unsigned long long)nq);
  }
}

// dst[seg..] = a*x[seg..] (+ b*y[seg..]) over len elements, for the active RHS
__global__ void k_lincomb(VecView dst, long long doff, VecView xv, long long xoff, double a, VecView yv,
                          long long yoff, double b, int use_y, long long len, const int* rmap, int nq) {
  const long long total = len * nq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / len);
    const long long i = e - (long long)q * len;
    const int r = rmap[q];
    double2 v = cscale(ld_cg(xv.p + r * xv.stride + xoff + i), a);
    if (use_y) v = cadd(v, cscale(ld_cg(yv.p + r * yv.stride + yoff + i), b));
    dst.p[r * dst.stride + doff + i] = v;
  }
}

// squared norms per active RHS: out[r] = sum |v|^2 (one CTA per RHS)
__global__ void k_norm2(VecView v, long long len, const int* rmap, double* out) {
  __shared__ double red[32];
  const int r = rmap[blockIdx.x];
  const double2* p = v.p + r * v.stride;
  double s = 0.0;
  for (long long i = threadIdx.x; i < len; i += blockDim.x) {
    const double2 a = p[i];
    s += a.x * a.x + a.y * a.y;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[r] = s;
}

// complex dots per active RHS: out[r] = vdot(x, y) = sum conj(x) y (one CTA per RHS, fixed-order sums)
__global__ void k_cdot(VecView x, VecView y, long long len, const int* rmap, double2* out) {
  __shared__ double red[64];
  const int r = rmap[blockIdx.x];
  const double2* a = x.p + r * x.stride;
  const double2* b = y.p + r * y.stride;
  double sr = 0.0, si = 0.0;
  for (long long i = threadIdx.x; i < len; i += blockDim.x) {
    const double2 c = cconjmul(ld_cg(a + i), ld_cg(b + i));
    sr += c.x;
    si += c.y;
  }
  const double2 h = block_sum2(sr, si, red);
  if (threadIdx.x == 0) out[r] = h;
}

// BiCGstab vector updates (krylov.py:164-196) per active RHS r with complex coefficients a[r], b[r]:
//   mode 0: d = x + a y              (s = r - alpha v with a = -alpha; r = s - omega t; x + alpha p)
//   mode 1: d = x + a (d - b y)      (p = r + beta (p - omega v))
//   mode 2: d = (d + a y) + b z      (x = x + alpha p + omega s)
__global__ void k_bicg_update(int mode, VecView d, VecView x, VecView y, VecView z, const double2* a,
                              const double2* b, long long len, const int* rmap, int nq) {
  const long long total = len * nq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / len);
    const long long i = e - (long long)q * len;
    const int r = rmap[q];
    double2* dp = d.p + r * d.stride + i;
    const double2 yv = ld_cg(y.p + r * y.stride + i);
    if (mode == 0) {
      *dp = cadd(ld_cg(x.p + r * x.stride + i), cmul(a[r], yv));
    } else if (mode == 1) {
      *dp = cadd(ld_cg(x.p + r * x.stride + i), cmul(a[r], csub(*dp, cmul(b[r], yv))));
    } else {
      *dp = cadd(cadd(*dp, cmul(a[r], yv)), cmul(b[r], ld_cg(z.p + r * z.stride + i)));
    }
  }
}

// dst = src / scale[r] (scale on device)
__global__ void k_scale_div(VecView dst, VecView src, long long len, const int* rmap, int nq,
                            const double* scale) {
  const long long total = len * nq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / len);
    const long long i = e - (long long)q * len;
    const int r = rmap[q];
    const double s = 1.0 / scale[r];  // one division per element instead of two
    const double2 a = src.p[r * src.stride + i];
    dst.p[r * dst.stride + i] = make_double2(a.x * s, a.y * s);
  }
}

// Fused MGS (krylov.py:89-94) for one RHS per CTA: for i = 0..j
//   h_i = vdot(V_i, w); w -= h_i V_i;   then hn = ||w||.
// V: [r][cap+1][n]; w is V_{j+1}.  hout[r][0..j] = h, hout[r][j+1] = hn.
__global__ void k_arnoldi(double2* V, long long vstride, long long n, int j, const int* rmap, double2* hout,
                          int hld) {
  __shared__ double red[32];
  const int r = rmap[blockIdx.x];
  double2* base = V + r * vstride;
  double2* w = base + (long long)(j + 1) * n;
  for (int i = 0; i <= j; ++i) {
    const double2* vi = base + (long long)i * n;
    double sr = 0.0, si = 0.0;
    for (long long e = threadIdx.x; e < n; e += blockDim.x) {
      const double2 c = cconjmul(vi[e], w[e]);
      sr += c.x;
      si += c.y;
    }
    sr = block_sum(sr, red);
    si = block_sum(si, red);
    const double2 h = make_double2(sr, si);
    for (long long e = threadIdx.x; e < n; e += blockDim.x) w[e] = csub(w[e], cmul(h, vi[e]));
    if (threadIdx.x == 0) hout[(size_t)r * hld + i] = h;
    __syncthreads();
  }
  double s = 0.0;
  for (long long e = threadIdx.x; e < n; e += blockDim.x) s += w[e].x * w[e].x + w[e].y * w[e].y;
  s = block_sum(s, red);
  if (threadIdx.x == 0) hout[(size_t)r * hld + j + 1] = make_double2(sqrt(s), 0.0);
}

// The same MGS step on a cluster of two CTAs per RHS (each owns half of the vector; the partial dots meet through
// distributed shared memory, summed rank 0 + rank 1 on both sides): the step is bound by per-SM bandwidth, and
// one CTA per RHS leaves most SMs idle for <= 74 RHS.  grid = 2 * active RHS.
__global__ void __cluster_dims__(2, 1, 1) k_arnoldi2(double2* V, long long vstride, long long n, int j,
                                                     const int* rmap, double2* hout, int hld) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double red[32];
  __shared__ double2 mine[2];  // this CTA's partial (re, im), double-buffered by step parity
  const int rank = (int)cl.block_rank();
  const int r = rmap[blockIdx.x >> 1];
  double2* base = V + r * vstride;
  double2* w = base + (long long)(j + 1) * n;
  const long long e0 = rank * (n / 2), e1 = rank == 0 ? n / 2 : n;
  const double2* peer = cl.map_shared_rank(mine, rank ^ 1);
  for (int i = 0; i <= j + 1; ++i) {  // i == j + 1: the norm of the orthogonalised vector
    const double2* vi = base + (long long)i * n;
    double sr = 0.0, si = 0.0;
    if (i <= j) {
      for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const double2 c = cconjmul(vi[e], w[e]);
        sr += c.x;
        si += c.y;
      }
    } else {
      for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) sr += w[e].x * w[e].x + w[e].y * w[e].y;
    }
    sr = block_sum(sr, red);
    si = block_sum(si, red);
    if (threadIdx.x == 0) mine[i & 1] = make_double2(sr, si);
    cl.sync();  // both partials are written (and the peer has finished reading the buffer of step i - 2)
    const double2 a = mine[i & 1], b = peer[i & 1];
    const double2 h = rank == 0 ? cadd(a, b) : cadd(b, a);  // rank 0's partial first on both CTAs
    if (i <= j) {
      for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) w[e] = csub(w[e], cmul(h, vi[e]));
      if (rank == 0 && threadIdx.x == 0) hout[(size_t)r * hld + i] = h;
    } else if (rank == 0 && threadIdx.x == 0) {
      hout[(size_t)r * hld + j + 1] = make_double2(sqrt(h.x), 0.0);
    }
  }
  cl.sync();  // no CTA exits while its shared memory may still be read
}

// x[r] += sum_i y[r][i] V[r][i]   (krylov.py:128-131)
__global__ void k_accum_x(VecView x, const double2* V, long long vstride, long long n, const double2* y,
                          int yld, int k, const int* rmap, int nq) {
  const long long total = n * nq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / n);
    const long long i = e - (long long)q * n;
    const int r = rmap[q];
    double2 acc = czero();
    for (int l = 0; l < k; ++l) cfma(acc, V[r * vstride + (long long)l * n + i], y[(size_t)r * yld + l]);
    double2* xp = x.p + r * x.stride + i;
    *xp = cadd(*xp, acc);
  }
}

// K5: ||H u - f||^2 and ||f||^2 per RHS (sie.py:441-445), 5-point PML stencil
__global__ void k_residual(const double2* u, const double2* f, long long stride, int wz, int wx, const double2* tx,
                           const double2* tz, const double* m, double omega2, const int* rmap, double* out,
                           const double2* hdiag) {
  __shared__ double red[32];
  const int r = rmap[blockIdx.y];
  const double2* ur = u + r * stride;
  const double2* fr = f + r * stride;
  double rr = 0.0, ff = 0.0;
  const long long N = (long long)wz * wx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / wx), pcol = (int)(e % wx);
    // diag = (Tx_main + Tz_main) - omega^2 m
    const double2 dg = hdiag ? hdiag[e] : csub(cadd(tx[wx + pcol], tz[wz + q]), make_double2(omega2 * m[e], 0.0));
    double2 a = cmul(dg, ur[e]);
    if (pcol > 0) a = cadd(a, cmul(tx[pcol], ur[e - 1]));
    if (pcol < wx - 1) a = cadd(a, cmul(tx[2 * wx + pcol], ur[e + 1]));
    if (q > 0) a = cadd(a, cmul(tz[q], ur[e - wx]));
    if (q < wz - 1) a = cadd(a, cmul(tz[2 * wz + q], ur[e + wx]));
    const double2 d = csub(a, fr[e]);
    rr += d.x * d.x + d.y * d.y;
    ff += fr[e].x * fr[e].x + fr[e].y * fr[e].y;
  }
  rr = block_sum(rr, red);
  ff = block_sum(ff, red);
  if (threadIdx.x == 0) {
    atomicAdd(out + 2 * r, rr);
    atomicAdd(out + 2 * r + 1, ff);
  }
}

// full-volume norms ||f||^2 per RHS (zero-source detection, sie.py:397-399)
// flags[l * R + r] = 1 when the split source of RHS r (sie.py:134-151: rows [off + lo, off + hi) of layer l) has a
// nonzero entry.  grid (L, R).
__global__ void k_slab_flags(const double2* f, long long stride, const LayerInfo* layers, int wx, int R, int* flags) {
  const LayerInfo& lay = layers[blockIdx.x];
  const int r = blockIdx.y;
  const double2* base = f + (size_t)r * stride + (size_t)(lay.off + lay.lo) * wx;
  const long long n = (long long)(lay.hi - lay.lo) * wx;
  int any = 0;
  for (long long e = threadIdx.x; e < n && !any; e += blockDim.x) {
    const double2 v = base[e];
    any |= v.x != 0.0 || v.y != 0.0;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) flags[blockIdx.x * R + r] = any;
}

__global__ void k_vol_norm2(const double2* f, long long stride, long long N, double* out) {
  __shared__ double red[32];
  const int r = blockIdx.y;
  double s = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x) {
    const double2 a = f[r * stride + e];
    s += a.x * a.x + a.y * a.y;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) atomicAdd(out + r, s);
}

// Green blocks, column-major [16 blocks][w cols][w rows] -> tile-major [16][ceil(w/8)][w][8]
// (rows >= w zero-padded), the layout the inner kernel streams with one bulk copy per tile.
// pass-0 operator rows: ABI order (4 w table rows, then (k, o) k-major) -> device order (q0_rows, pt_device.cuh)
__global__ void k_q0_rows(const double2* src, double2* dst, int w, int nk, int K) {
  const int tab8 = q0_tab8(w), nk8 = q0_nk8(nk);
  const long long tot = (long long)q0_rows(w, nk) * K;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(e / K), k = (int)(e - (long long)m * K);
    long long srow = -1;
    if (m < 4 * w) {
      srow = m;
    } else if (m >= tab8) {
      const int mm = m - tab8, oi = mm / nk8, kk = mm - oi * nk8;
      if (kk < nk) srow = 4LL * w + 4LL * kk + oi;
    }
    dst[e] = srow >= 0 ? src[srow * K + k] : make_double2(0.0, 0.0);
  }
}

// C = A B for 2 x 2 block matrices of column-major w x w blocks ([s][k][w*w]; element (i, j) of a block at
// j * w + i): C[s][k] = sum_m A[s][m] B[m][k].  Offline products of the scan-form inner sweeps (solver.cu).
// grid (ceil(w/16), ceil(w/16), 4), block (16, 16).
__global__ void k_block2_mm(const double2* A, const double2* B, double2* C, int w) {
  __shared__ double2 as[16][17], bs[16][17];
  const int sb = blockIdx.z >> 1, kb = blockIdx.z & 1;
  const int i = blockIdx.x * 16 + threadIdx.x, j = blockIdx.y * 16 + threadIdx.y;
  const size_t W = (size_t)w * w;
  double2 acc = make_double2(0.0, 0.0);
  for (int m = 0; m < 2; ++m) {
    const double2* Ab = A + (size_t)(sb * 2 + m) * W;
    const double2* Bb = B + (size_t)(m * 2 + kb) * W;
    for (int t0 = 0; t0 < w; t0 += 16) {
      const int ta = t0 + threadIdx.y, tb = t0 + threadIdx.x;
      as[threadIdx.y][threadIdx.x] = (i < w && ta < w) ? Ab[(size_t)ta * w + i] : make_double2(0.0, 0.0);
      bs[threadIdx.y][threadIdx.x] = (tb < w && j < w) ? Bb[(size_t)j * w + tb] : make_double2(0.0, 0.0);
      __syncthreads();
#pragma unroll
      for (int t = 0; t < 16; ++t) cfma(acc, as[t][threadIdx.x], bs[threadIdx.y][t]);
      __syncthreads();
    }
  }
  if (i < w && j < w) C[(size_t)(sb * 2 + kb) * W + (size_t)j * w + i] = acc;
}

__global__ void k_green_tiles(const double2* src, double2* dst, int w, int nb) {
  const int nmt = (w + 7) >> 3;
  const long long total = (long long)nb * nmt * w * 8;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e & 7);
    long long rest = e >> 3;
    const int k = (int)(rest % w);
    rest /= w;
    const int mt = (int)(rest % nmt);
    const int b = (int)(rest / nmt);
    const int i = mt * 8 + r;
    dst[e] = i < w ? src[((size_t)b * w + k) * w + i] : make_double2(0.0, 0.0);
  }
}

// dense inner operator (row-major n x n) -> DMMA fragments, chunk-major: [chunk c of kc k-steps][8-row tile t]
// [k-step kl < kc][32 lanes], lane = 4 r + col holding M[8 t + r][4 (c kc + kl) + col] (zero past n or past the
// last k-step), so the tiles [t0, t1) of one chunk are one contiguous bulk copy
// three n x n row-major matrices stacked by row tiles in the dense fragment layout: [chunk][3 T8][kc][32]
__global__ void k_dense_tiles_stack3(const double2* s0, const double2* s1, const double2* s2, double2* dst, int n,
                                     int kc) {
  const int T8 = (n + 7) >> 3, nks = n >> 2, nch = (nks + kc - 1) / kc;
  const long long total = (long long)nch * 3 * T8 * kc * 32;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(e & 31);
    long long rest = e >> 5;
    const int kl = (int)(rest % kc);
    rest /= kc;
    const int ts = (int)(rest % (3 * T8)), c = (int)(rest / (3 * T8));
    const int m = ts / T8, t = ts - m * T8;
    const double2* src = m == 0 ? s0 : (m == 1 ? s1 : s2);
    const int row = t * 8 + (lane >> 2), ks = c * kc + kl, k = ks * 4 + (lane & 3);
    dst[e] = (row < n && ks < nks) ? src[(size_t)row * n + k] : make_double2(0.0, 0.0);
  }
}

__global__ void k_dense_tiles(const double2* src, double2* dst, int n, int kc) {
  const int T8 = (n + 7) >> 3, nks = n >> 2, nch = (nks + kc - 1) / kc;
  const long long total = (long long)nch * T8 * kc * 32;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(e & 31);
    long long rest = e >> 5;
    const int kl = (int)(rest % kc);
    rest /= kc;
    const int t = (int)(rest % T8), c = (int)(rest / T8);
    const int row = t * 8 + (lane >> 2), ks = c * kc + kl, k = ks * 4 + (lane & 3);
    dst[e] = (row < n && ks < nks) ? src[(size_t)row * n + k] : make_double2(0.0, 0.0);
  }
}

// ---------------------------------------------------------------------------------------------
// Sampled trace-source response (replaces the second cell-solve pass of a layer solve whose only
// outputs are layer-row samples).  By linearity the reconstruction-pass solution is
//   u1 = H_c^{-1}(f + panels) + sum_s H_c^{-1}(coef_s E_krow_s) tr_s = u0 + sum_s G_s tr_s,
// so its samples at the layer trace rows are the pass-0 samples (written by K1 pass 0) plus
// gsmp[k][row][s][:] . tr_s for every kept block row k.
// grid: x = job * Lc + cell, y = group of 8 RHS, z = chunk of kept block rows.
cudaError_t green_samples_launch(const OJob* jobs, int J, const CellInfo* cells, const LayerInfo* layers,
                                 const double2* gsmp, const double2* tr, double2* smp, int R, int Lc, int wx,
                                 int wmax, int kmax, int num_sms, cudaStream_t st, const VecTab* tab,
                                 const int* rmap) {
  const int fuse_combine = tab != nullptr;
  const VecTab tabv = tab ? *tab : VecTab{};
  if (J == 0 || R == 0) return cudaSuccess;
  if (R >= stage_gemm_min_cols(0))  // the streaming tensor-core GEMM (stage_gemm.cu)
    return sample_gemm_launch(jobs, J, cells, layers, gsmp, tr, smp, R, Lc, wx, wmax, kmax, num_sms, st, tab, rmap);
  const int gy = (R + 7) / 8;
  // rows per cell <= kmax kept block rows x 4 output rows; one 8-row tile per warp
  const int gz = (kmax * 4 + 8 * GS_WARPS - 1) / (8 * GS_WARPS);
  static const bool v1 = std::getenv("PT_GS_V1") != nullptr;
  if (v1) {
    const size_t sm = sizeof(double2) * 4 * (size_t)((wmax + 3) & ~3) * 8;
    if (sm > 48 * 1024) set_smem_attr((const void*)k_green_samples, sm);
    k_green_samples<<<dim3(J * Lc, gy, gz), GS_WARPS * 32, sm, st>>>(jobs, cells, layers, gsmp, tr, smp, R, Lc, wx, wmax,
                                                                          tabv, rmap, fuse_combine);
    return cudaGetLastError();
  }
  const int gy2 = (R + 8 * GS2_NG - 1) / (8 * GS2_NG);
  const int gz2 = (kmax * 4 + 8 * GS2_TPC - 1) / (8 * GS2_TPC);
  const size_t sm2 = sizeof(double2) * 4 * (size_t)((wmax + 3) & ~3) * 8 * GS2_NG +
                     sizeof(double) * GS2_TPC * (GS2_KQ - 1) * GS2_NG * 4 * 32;
  if (sm2 > 48 * 1024) set_smem_attr((const void*)k_green_samples2, sm2);
  k_green_samples2<<<dim3(J * Lc, gy2, gz2), GS2_KQ * GS2_TPC * 32, sm2, st>>>(jobs, cells, layers, gsmp, tr, smp, R, Lc,
                                                                               wx, wmax, tabv, rmap, fuse_combine);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// First pass of a layer solve without a volume source, as one dense product per cell:
//   out[m][n] = sum_{s,k} Q0[m][(s,k)] * P[job(n)][s][q(n)][off_c + lo + k]
// m < 4w: Newton-table rows (block row r0/r1/rn/rnp, column j); m >= 4w: layer-row samples
// (kept block row k, row 0/1/n/n+1).  DMMA m8n8k4 f64 complex (4 products per k-step), one 8-row
// tile x up to 32 columns (4 groups of 8) per warp, A from the operator pool, B from the gathered panels.
// grid: x = layer group g * Lc + cell, y = chunk of 8 row tiles, z = chunk of 32 columns.
cudaError_t pass0_launch(const int* grp, int ngroups, const int* ljobs, const OJob* jobs, const CellInfo* cells,
                         const LayerInfo* layers, const double2* q0, const double2* P, double2* tables, double2* smp,
                         int R, int Lc, int wx, int wmax, int kmax, int max_jobs_per_layer, cudaStream_t st,
                         int accum, const VecTab* tab, const int* rmap, const RhsOut* rhs_out) {
  if (ngroups == 0 || R == 0) return cudaSuccess;
  if (!tab && max_jobs_per_layer * R >= stage_gemm_min_cols(1)) {  // many columns: stage_gemm.cu
    static int nsm = 0;
    if (!nsm) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    return pass0_gemm_launch(grp, ngroups, ljobs, jobs, cells, layers, q0, P, tables, smp, R, Lc, wx, wmax, kmax,
                             max_jobs_per_layer, nsm, st, accum, rhs_out);
  }
  const VecTab tabv = tab ? *tab : VecTab{};
  const int mp = q0_rows(wmax, kmax);
  const int gz = (max_jobs_per_layer * R + P0_COLS - 1) / P0_COLS;
  const RhsOut ro = rhs_out ? *rhs_out : RhsOut{nullptr, 0, 0};
  // k-loop variant: (slot, k) advanced incrementally across the used slots (default) or per-slot segments with
  // contiguous addresses (PT_P0_SEG=1; measured 4 % slower on cfg2: 9.80-10.05 vs 9.39-9.51 ms per step)
  static const bool no_seg = std::getenv("PT_P0_SEG") == nullptr;
  if (tab)
    k_pass0<true, true><<<dim3(ngroups * Lc, mp / 8, gz), P0_KQ * 32, 0, st>>>(grp, ljobs, jobs, cells, layers, q0, P, tables,
                                                                       smp, R, Lc, wx, wmax, accum, tabv, rmap, 1, ro);
  else if (no_seg)
    k_pass0<false, false><<<dim3(ngroups * Lc, mp / 8, gz), P0_KQ * 32, 0, st>>>(grp, ljobs, jobs, cells, layers, q0, P,
                                                                               tables, smp, R, Lc, wx, wmax, accum, tabv,
                                                                               rmap, 0, ro);
  else
    k_pass0<false, true><<<dim3(ngroups * Lc, mp / 8, gz), P0_KQ * 32, 0, st>>>(grp, ljobs, jobs, cells, layers, q0, P,
                                                                              tables, smp, R, Lc, wx, wmax, accum, tabv,
                                                                              rmap, 0, ro);
  return cudaGetLastError();
}
