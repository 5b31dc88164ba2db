// Device bodies of the stage kernels (gather, pass-0 product, sampled trace response, combine), shared by
// the standalone kernels (outer_kernels.cu) and the fused cooperative stage kernel (inner_gmres.cu).
#pragma once
#include "pt_launch.cuh"

__device__ __forceinline__ double2 vref(const VecTab& t, Ref rf, int r, int x, int wx) {
  return ld_cg(t.v[rf.vec].p + (size_t)r * t.v[rf.vec].stride + (size_t)rf.seg * wx + x);
}

// P[job][s][q][x] = sum of the slot's refs (sie.py:203-308 panel expressions); one element e
__device__ __forceinline__ void gather_elem(const OJob* jobs, const VecTab& t, const int* rmap, int nq, int wx,
                                            double2* P, long long e) {
  const int x = (int)(e % wx);
  long long rest = e / wx;
  const int q = (int)(rest % nq);
  rest /= nq;
  const int s = (int)(rest % 4);
  const int j = (int)(rest / 4);
  const Ref* pr = jobs[j].pan[s];
  if (pr[0].vec < 0) {  // absent slot: zero (the dense pass-0 product reads every slot)
    P[e] = make_double2(0.0, 0.0);
    return;
  }
  const int r = rmap[q];
  double2 v = vref(t, pr[0], r, x, wx);
  if (pr[1].vec >= 0) v = cadd(v, vref(t, pr[1], r, x, wx));
  P[e] = v;
}

// dst = scoef*sample + add - (sub0 + sub1); one element e of [job][4][q][x]
__device__ __forceinline__ void combine_elem(const OJob* jobs, const VecTab& t, const int* rmap, int nq, int wx,
                                             const double2* smp, long long e) {
  const int x = (int)(e % wx);
  long long rest = e / wx;
  const int q = (int)(rest % nq);
  rest /= nq;
  const int o = (int)(rest % 4);
  const int j = (int)(rest / 4);
  const OJob& jb = jobs[j];
  if (o >= jb.nout) return;
  const int r = rmap[q];
  double2 y = cscale(smp[e], jb.scoef[o]);
  if (jb.add[o].vec >= 0) y = cadd(y, vref(t, jb.add[o], r, x, wx));
  if (jb.sub[o][0].vec >= 0) {
    double2 sb = vref(t, jb.sub[o][0], r, x, wx);
    if (jb.sub[o][1].vec >= 0) sb = cadd(sb, vref(t, jb.sub[o][1], r, x, wx));
    y = csub(y, sb);
  }
  const VecView& dv = t.v[jb.dst[o].vec];
  dv.p[(size_t)r * dv.stride + (size_t)jb.dst[o].seg * wx + x] = y;
}

#define P0_COLS 16  // columns (job, RHS) per CTA: two DMMA column groups of 8
#ifndef P0_KQ
#define P0_KQ 4      // k parts per row tile (one warp each), summed in shared memory in a fixed order
#endif
// One (layer group g, cell c, row tile, 16-column chunk z) item, executed by P0_KQ warps (wq = warp index in
// the group); part: [P0_KQ-1][2][4][32] doubles of shared memory; barid: named barrier of the group;
// accum: add to the Newton tables instead of overwriting them.
template <bool DIRECT = false, bool SEG = true>
__device__ __forceinline__ void pass0_item(const int* __restrict__ grp, const int* __restrict__ ljobs,
                                           const OJob* __restrict__ jobs, const CellInfo* __restrict__ cells,
                                           const LayerInfo* __restrict__ layers, const double2* __restrict__ q0,
                                           const double2* __restrict__ P, double2* __restrict__ tables,
                                           double2* __restrict__ smp, int R, int Lc, int wx, int wmax, int g, int c,
                                           int tile, int z, int wq, double* part, int barid, int accum = 0,
                                           const VecTab* tabd = nullptr, const int* rmap = nullptr,
                                           const RhsOut* rhs_out = nullptr) {
  const int layer = grp[3 * g], jb0 = grp[3 * g + 1], nj = grp[3 * g + 2];
  const CellInfo& ci = cells[layer * Lc + c];
  const LayerInfo& lay = layers[layer];
  const int w = ci.w, nk = ci.hi - ci.lo, nk4 = (nk + 3) & ~3, K = 4 * nk4;
  const int tab8 = q0_tab8(w), nk8 = q0_nk8(nk), Mp = tab8 + 4 * nk8;  // device row layout (pt_device.cuh)
  const int lane = threadIdx.x & 31, wp = wq;
  const int N = nj * R, n0 = z * P0_COLS;
  if (n0 >= N || tile * 8 >= Mp) return;
  if (tile * 8 >= tab8) {  // a sample tile of output row oi: skipped when no job of these columns samples that row
    const int oi_t = (tile * 8 - tab8) / nk8;
    bool need = false;
    for (int jj = n0 / R; jj < nj && jj * R < n0 + P0_COLS; ++jj) {
      const OJob& jo = jobs[ljobs[jb0 + jj]];
      for (int o = 0; o < jo.nout; ++o) {
        const int orow = jo.orow[o];
        need |= (orow == 0 ? 0 : (orow == 1 ? 1 : (orow == lay.n ? 2 : 3))) == oi_t;
      }
    }
    if (!need) return;
  }
  const int ngq = min(2, (N - n0 + 7) >> 3);
  const int ar = lane >> 2, ak = lane & 3;
  const double2* arow = q0 + ci.q0_off + (size_t)(tile * 8 + ar) * K + ak;
  const double2* bcol[2];
  bool bok[2];
  int jidg[2], rg[2];
#pragma unroll
  for (int gq = 0; gq < 2; ++gq) {
    const int n = n0 + 8 * gq + ar;
    bok[gq] = n < N;
    const int jid = ljobs[jb0 + (bok[gq] ? n / R : 0)], q = bok[gq] ? n % R : 0;
    jidg[gq] = jid;
    rg[gq] = tabd ? rmap[q] : 0;
    bcol[gq] = P + ((size_t)(jid * 4) * R + q) * wx + ci.off + ci.lo + ak;
  }
  const size_t sstride = (size_t)R * wx;  // slot stride in P
  // B element: the gathered panel P, or (tabd) the panel sum read straight from the outer vectors
  auto bload = [&](int gq, int sl, int kk) -> double2 {
    if constexpr (!DIRECT) return __ldg(bcol[gq] + sl * sstride + kk);
    const Ref ra = jobs[jidg[gq]].pan[sl][0], rb = jobs[jidg[gq]].pan[sl][1];
    const int x = ci.off + ci.lo + kk + ak;
    double2 v = ra.vec >= 0 ? vref(*tabd, ra, rg[gq], x, wx) : make_double2(0.0, 0.0);
    if (rb.vec >= 0) v = cadd(v, vref(*tabd, rb, rg[gq], x, wx));
    return v;
  };
  double acc[2][4];
#pragma unroll
  for (int gq = 0; gq < 2; ++gq) acc[gq][0] = acc[gq][1] = acc[gq][2] = acc[gq][3] = 0.0;
  // only the slots some job of this layer group feeds (absent slot panels are zero): the K range runs over
  // the used slots, packed (sweep stages use 1-2 of the 4)
  int slist = 0, nsl = 0;
  {
    int used = 0;
    for (int jj = 0; jj < nj; ++jj) {
      const OJob& jo = jobs[ljobs[jb0 + jj]];
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) used |= (jo.pan[sl][0].vec >= 0) << sl;
    }
#pragma unroll
    for (int sl = 0; sl < 4; ++sl)
      if (used >> sl & 1) slist |= sl << (2 * nsl++);
  }
  const int kps = nk4 >> 2, nks = nsl * kps;  // k-steps per slot / over the used slots
  const int kb = wp * nks / P0_KQ, ke = (wp + 1) * nks / P0_KQ;
  if constexpr (SEG) {
  // the warp's k-steps [kb, ke) as per-slot segments: contiguous A and B addresses inside a segment
  for (int si = kps > 0 ? kb / kps : nsl; si < nsl && si * kps < ke; ++si) {
    const int sl = slist >> (2 * si) & 3;
    const int r0 = max(kb - si * kps, 0), r1 = min(ke - si * kps, kps);  // k-steps [r0, r1) of this slot
    const double2* ap = arow + (size_t)(sl * kps + r0) * 4;
    const double2* bp0 = bcol[0] + sl * sstride;
    const double2* bp1 = bcol[1] + sl * sstride;
    for (int rs = r0; rs < r1; rs += 8) {
      double2 av[8], bv[8][2];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int rr = rs + u, kk = rr * 4;
        const bool kin = rr < r1;
        av[u] = kin ? __ldg(ap + (size_t)(rr - r0) * 4) : make_double2(0.0, 0.0);
        const bool kok = kin && kk + ak < nk;
        if constexpr (DIRECT) {
          bv[u][0] = (kok && bok[0]) ? bload(0, sl, kk) : make_double2(0.0, 0.0);
          bv[u][1] = (kok && bok[1]) ? bload(1, sl, kk) : make_double2(0.0, 0.0);
        } else {
          bv[u][0] = (kok && bok[0]) ? __ldg(bp0 + kk) : make_double2(0.0, 0.0);
          bv[u][1] = (kok && bok[1]) ? __ldg(bp1 + kk) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
#pragma unroll
        for (int gq = 0; gq < 2; ++gq) {
          if (gq < ngq) {
            dmma_f64(acc[gq][0], acc[gq][1], av[u].x, bv[u][gq].x);
            dmma_f64(acc[gq][2], acc[gq][3], av[u].x, bv[u][gq].y);
            dmma_f64(acc[gq][0], acc[gq][1], -av[u].y, bv[u][gq].y);
            dmma_f64(acc[gq][2], acc[gq][3], av[u].y, bv[u][gq].x);
          }
        }
      }
    }
  }
  } else {
  // (used-slot index, k-step within the slot) of the next k-step, advanced incrementally (no divisions)
  int si_c = kps > 0 ? kb / kps : 0, r_c = kb - si_c * kps;
  for (int ks0 = kb; ks0 < ke; ks0 += 8) {
    double2 av[8], bv[8][2];
    int si = si_c, r = r_c;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool kin = ks0 + u < ke;
      const int sl = slist >> (2 * (si & 3)) & 3;
      const int kk = r * 4;  // column within the slot block (+ ak)
      av[u] = kin ? __ldg(arow + (sl * kps + r) * 4) : make_double2(0.0, 0.0);
#pragma unroll
      for (int gq = 0; gq < 2; ++gq)
        bv[u][gq] = (kin && bok[gq] && kk + ak < nk) ? bload(gq, sl, kk) : make_double2(0.0, 0.0);
      if (++r == kps) {
        r = 0;
        ++si;
      }
    }
    si_c = si;
    r_c = r;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int gq = 0; gq < 2; ++gq) {
        if (gq < ngq) {
          dmma_f64(acc[gq][0], acc[gq][1], av[u].x, bv[u][gq].x);
          dmma_f64(acc[gq][2], acc[gq][3], av[u].x, bv[u][gq].y);
          dmma_f64(acc[gq][0], acc[gq][1], -av[u].y, bv[u][gq].y);
          dmma_f64(acc[gq][2], acc[gq][3], av[u].y, bv[u][gq].x);
        }
      }
    }
  }
  }
  if (wp > 0) {
#pragma unroll
    for (int gq = 0; gq < 2; ++gq)
#pragma unroll
      for (int t = 0; t < 4; ++t) part[(((wp - 1) * 2 + gq) * 4 + t) * 32 + lane] = acc[gq][t];
  }
  named_bar(barid, P0_KQ * 32);
  if (wp > 0) return;
#pragma unroll
  for (int p2 = 0; p2 < P0_KQ - 1; ++p2)
#pragma unroll
    for (int gq = 0; gq < 2; ++gq)
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[gq][t] += part[((p2 * 2 + gq) * 4 + t) * 32 + lane];
  // C fragment: row ar of the tile, columns 2 ak, 2 ak + 1 of each group
  const int m = tile * 8 + ar;
  if (m >= 4 * w && (m < tab8 || (m - tab8) % nk8 >= nk)) return;  // padding rows
#pragma unroll
  for (int gq = 0; gq < 2; ++gq) {
    if (gq >= ngq) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = n0 + 8 * gq + 2 * ak + h;
      if (n >= N) continue;
      const int jid = ljobs[jb0 + n / R], q = n % R;
      const double2 v = make_double2(acc[gq][h], acc[gq][2 + h]);
      if (m < 4 * w) {
        const int idx = m / w, j = m - (m / w) * w;
        double2* tp = tables + ((((size_t)jid * Lc + c) * 4 + idx) * R + q) * wmax + j;
        const double2 tv = accum ? cadd(*tp, v) : v;
        *tp = tv;
        if (rhs_out) {  // rows n, n+1 of cell c < nI feed down[c]; rows 0, 1 of cell c >= 1 feed up[c - 1]
          const int nIc = Lc - 1;
          int seg = -1;
          if (idx >= 2 && c < nIc) seg = 2 * c + (idx - 2);
          else if (idx < 2 && c >= 1) seg = 2 * nIc + 2 * (c - 1) + idx;
          if (seg >= 0)
            rhs_out->base[((size_t)jid * R + q) * rhs_out->stride + rhs_out->off + (size_t)seg * w + j] =
                make_double2(-tv.x, -tv.y);
        }
      } else {
        const int mm = m - tab8, oi = mm / nk8, kk = mm - oi * nk8;
        const OJob& jb = jobs[jid];
        for (int o = 0; o < jb.nout; ++o) {
          const int orow = jb.orow[o];
          const int ok_ = orow == 0 ? 0 : (orow == 1 ? 1 : (orow == lay.n ? 2 : 3));
          if (ok_ == oi) smp[((size_t)(jid * 4 + o) * R + q) * wx + ci.off + ci.lo + kk] = v;
        }
      }
    }
  }
}


// DMMA formulation: rows = (kept block row k, output row o) of a cell, N = 8 RHS, K = (slot, column j):
//   C[(k,o)][r] += sum_{s,j} G[k][o][s][j] * tr_s[r][j]   (complex: Cr += Ar Br - Ai Bi, Ci += Ar Bi + Ai Br)
// A fragments straight from the sampled Green pool (each element used once per CTA), B fragments from the
// trace panels staged in shared memory as [slot][j (padded to w4, zeros)][8 RHS]; one 8-row tile per warp.
#define GS_WARPS 8
// One (job x cell, 8-RHS group y, kept-row chunk z of gz) item, executed by a whole CTA of GS_WARPS warps;
// trs: [4 slots][w4][8 rhs] shared memory (4 * roundup(wmax,4) * 8 double2).
__device__ __forceinline__ void green_item(const OJob* __restrict__ jobs, const CellInfo* __restrict__ cells,
                                           const LayerInfo* __restrict__ layers, const double2* __restrict__ gsmp,
                                           const double2* __restrict__ tr, double2* __restrict__ smp, int R, int Lc,
                                           int wx, int wmax, int x, int y, int z, double2* trs,
                                           const VecTab* tabd = nullptr, const int* rmap = nullptr) {
  __syncthreads();  // trs of the previous item consumed
  const int jid = x / Lc, c = x - (x / Lc) * Lc;
  const OJob& jb = jobs[jid];
  const int nout = jb.nout;
  if (nout <= 0) return;
  const LayerInfo& lay = layers[jb.layer];
  const CellInfo& ci = cells[jb.layer * Lc + c];
  const int w = ci.w, w4 = (w + 3) & ~3, nIc = Lc - 1, tid = threadIdx.x;
  const int lane = tid & 31, wp = tid >> 5;
  const int r0 = y * 8, nr = min(8, R - r0);
  for (int row = wp; row < 32; row += GS_WARPS) {  // (slot, rhs) rows of the trace panels
    const int sl = row >> 3, rr = row & 7;
    const int I = sl < 2 ? c - 1 : c;
    const bool okr = rr < nr && I >= 0 && I < nIc;
    const double2* src = tr + (((size_t)(jid * R + r0 + (okr ? rr : 0)) * nIc + (okr ? I : 0)) * 2 + (sl & 1)) * wmax;
    for (int j = lane; j < w4; j += 32)
      trs[((size_t)sl * w4 + j) * 8 + rr] = (okr && j < w) ? src[j] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int s_lo = ci.has_top ? 0 : 2, s_hi = ci.has_bot ? 4 : 2;
  const int nrows = (ci.hi - ci.lo) * nout;  // (k, o) rows of this cell, k-major
  const int tile = z * GS_WARPS + wp;
  if (tile * 8 >= nrows) return;
  const int ar = lane >> 2, ak = lane & 3;
  // this lane's A row
  const int m = tile * 8 + ar;
  const bool mok = m < nrows;
  const int mk = mok ? m / nout : 0, mo = mok ? m - (m / nout) * nout : 0;
  const int orow = jb.orow[mo];
  const int oi = orow == 0 ? 0 : (orow == 1 ? 1 : (orow == lay.n ? 2 : 3));
  const double2* grow = gsmp + ci.gsmp_off + ((size_t)(ci.lo + mk) * 4 + oi) * 4 * w;  // [4 slots][w]
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  for (int sl = s_lo; sl < s_hi; ++sl) {
    const double2* ga = grow + sl * w;
    const double2* tb = trs + (size_t)sl * w4 * 8 + ar;
#pragma unroll 6
    for (int j0 = 0; j0 < w4; j0 += 4) {
      const int j = j0 + ak;
      const double2 av = (mok && j < w) ? __ldg(ga + j) : make_double2(0.0, 0.0);
      const double2 bv = tb[(size_t)j * 8];
      dmma_f64(c0, c1, av.x, bv.x);
      dmma_f64(c2, c3, av.x, bv.y);
      dmma_f64(c0, c1, -av.y, bv.y);
      dmma_f64(c2, c3, av.y, bv.x);
    }
  }
  // C fragment: row ar, columns (RHS) 2 ak and 2 ak + 1; (c0, c2) and (c1, c3) are complex
  if (!mok) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int rr = 2 * ak + h;
    if (rr < nr) {
      double2* dst = smp + ((size_t)(jid * 4 + mo) * R + r0 + rr) * wx + ci.off + ci.lo + mk;
      const double2 yv = cadd(*dst, h == 0 ? make_double2(c0, c2) : make_double2(c1, c3));
      if (!tabd) {
        *dst = yv;
      } else {  // combine fused in: out = scoef*sample + add - (sub0 + sub1) (k_combine)
        const int xg = ci.off + ci.lo + mk, r = rmap[r0 + rr];
        double2 o = cscale(yv, jb.scoef[mo]);
        if (jb.add[mo].vec >= 0) o = cadd(o, vref(*tabd, jb.add[mo], r, xg, wx));
        if (jb.sub[mo][0].vec >= 0) {
          double2 sb = vref(*tabd, jb.sub[mo][0], r, xg, wx);
          if (jb.sub[mo][1].vec >= 0) sb = cadd(sb, vref(*tabd, jb.sub[mo][1], r, xg, wx));
          o = csub(o, sb);
        }
        const VecView& dv = tabd->v[jb.dst[mo].vec];
        dv.p[(size_t)r * dv.stride + (size_t)jb.dst[mo].seg * wx + xg] = o;
      }
    }
  }
}

