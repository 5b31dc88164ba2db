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
#include <cstdio>

#include <cstdlib>
#include "pt_launch.cuh"

#ifndef K1_FETCH_POS
#define K1_FETCH_POS 0  // where the next step's operands are fetched: 0 before the matvec
#endif

namespace cg = cooperative_groups;

struct ColInfo {
  int jid, r, panmask, vol, nout, vfull, opos[4], pad[6];
};

// partial-sum sets of the matvec: DMMA path (NC == 8) splits k by parity, DFMA path by warp
// rows of the partial-sum area: one [w][NC] set per consumer warp
__host__ __device__ constexpr int k1_red_rows(int w) { return 7 * w; }

// Per-element descriptor of K1 (see the consumer section): base pointers of the per-step operands.
// 32-bit element offsets (-1 = absent) keep it at 24 bytes so the shared-memory ring stays large.
struct Desc {
  int pb;                // into P (panel source; coefficient = layer coef[slot])
  int vb;                // into f (passes 0/1) or the dense test rhs (pass 2)
  int tt, tbm;           // into tr: cell trace sources above / below (reconstruction pass)
  int ob;                // into the output array selected by okind
  unsigned char slot;    // panel slot of pb
  unsigned char okind;   // 0 none, 1 Newton tables, 2 volume u, 3 sampled smp, 4 dense test xd
  unsigned char pad[2];
  int ob2;               // pass 0 with s0: into smp (layer-row sample of the pass-0 solution), -1 none
};

template <int NC, int NMT>
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
  if (p.pass == 0 && p.zflag) {
    // every column of the task solves H_c x = 0 (zero split source, no panels): the outputs are zero
    bool allzero = true;
    for (int ql = 0; ql < task.nq && allzero; ++ql) {
      const int q = task.q0 + ql;
      const OJob& jb = p.jobs[p.ljobs[task.jb + q / p.R]];
      bool pans = false;
      for (int s = 0; s < 4; ++s) pans |= jb.pan[s][0].vec >= 0;
      allzero = !pans && jb.vol && !jb.vfull && p.zflag[jb.layer * p.R + q % p.R] == 0;
    }
    if (allzero) {  // uniform over the cluster (same task, same flags): nobody reaches a cluster barrier
      if (rank == 0) {
        const int nk = cell.hi - cell.lo;
        for (int ql = 0; ql < task.nq; ++ql) {
          const int q = task.q0 + ql, jid = p.ljobs[task.jb + q / p.R], r = q % p.R;
          const OJob& jb = p.jobs[jid];
          for (int e = tid; e < 4 * w; e += blockDim.x) {
            const int idx = e / w, j = e - idx * w;
            if (idx < 2 ? cell.has_top : cell.has_bot)
              p.tables[((size_t)(jid * p.Lc + cell.cell) * 4 + idx) * p.R * p.wmax + (size_t)r * p.wmax + j] = czero();
          }
          if (p.s0 && jb.nout > 0)
            for (int e = tid; e < jb.nout * nk; e += blockDim.x) {
              const int o = e / nk, k = e - o * nk;
              p.smp[((size_t)(jid * 4 + o) * p.R + r) * p.wx + cell.off + cell.lo + k] = czero();
            }
        }
      }
      return;
    }
  }
  const int NS = p.ns;  // ring slots (<= K1_NS; a multiple of CM)
  // elements (row, column) per consumer thread: w*NC <= (NC == 8 ? 8*NMT : 32*NMT) * NC
  constexpr int TT = ((NC == 8 ? 8 * NMT : 32 * NMT) * NC + K1_CONSUMERS - 1) / K1_CONSUMERS;
  const int nIc = p.Lc - 1;

  unsigned char* ring = smem;
  double2* VA = reinterpret_cast<double2*>(ring + (size_t)NS * p.slot_bytes);  // slot_bytes % 128 == 0
  const int w4v = (w + 3) & ~3;
  double2* VB = VA + w4v * NC;
  double2* XC = VB + w4v * NC;  // partner's half-chain vector at the middle block
  double2* red = XC + w4v * NC;
  ColInfo* cols = reinterpret_cast<ColInfo*>(red + k1_red_rows(w) * NC);
  uint64_t* full = reinterpret_cast<uint64_t*>(cols + NC);
  uint64_t* lempty = full + K1_NS;
  uint64_t* cempty = lempty + K1_NS;
  uint64_t* xbar = cempty + K1_NS;

  const int w4 = (w + 3) & ~3;  // stored columns per block (zero padded)
  const int jc = NC == 8 ? p.jc8 : 7 * k1_jw(NC);  // columns per ring chunk
  const int wcols = NC == 8 ? w4 : w;                // streamed columns (DMMA: zero padded to w4)
  const int nch = (wcols + jc - 1) / jc;
  const int total = nst * nch;
  const double2* S = p.sinv + cell.sinv_off;
  // factor block used by step s of this half
  auto kblk = [&](int s) -> int {
    if (h == 0) return s <= m ? s : 2 * m - s;
    return s < mb ? wzc - 1 - s : (s == mb ? m : m + (s - mb));
  };

  for (int e = tid; e < 2 * w4v * NC; e += blockDim.x) VA[e] = czero();
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
    for (int s = 0; s < K1_NS; ++s) {
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
      int slot = 0;
      uint32_t ph = 0;  // parity of the current use of `slot`
      for (int c = 0; c < total && !(p.dbg & 1); ++c) {
        const bool reuse = c >= NS;
        if (reuse) mbar_wait_suspend(&lempty[slot], ph ^ 1u);
        const int s = c / nch, ch = c - s * nch;
        const int c0 = ch * jc, cw = min(jc, wcols - c0);
        const uint32_t bytes = (uint32_t)cw * w * 16u;
        mbar_expect_tx(&full[slot], bytes);
        const int issuer = slot % CM;
        const double2* src = S + (size_t)kblk(s) * w * w4 + (size_t)c0 * w;
        unsigned char* dst = ring + (size_t)slot * p.slot_bytes;
        if (CM == 1) {
          bulk_g2s(dst, src, bytes, &full[slot]);
        } else {
          if (reuse) mbar_arrive_remote(mapa(&cempty[slot], (uint32_t)(h * CM + issuer)));
          if (issuer == cm) {
            if (reuse) mbar_wait(&cempty[slot], ph ^ 1u);
            bulk_g2s_mc(dst, src, bytes, &full[slot], mask);
          }
        }
        if (++slot == NS) {
          slot = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const int lane = tid & 31, wp = tid >> 5;
    double2* Z = p.Z + task.zoff + (size_t)cm * wzc * w * NC;
    const int nel = w * NC;
    const int partner = (1 - h) * CM + cm;
    auto kind_of = [&](int s) -> int {
      return (h == 0) ? (s < m ? 0 : (s == m ? 1 : 2)) : (s < mb ? 0 : (s == mb ? 1 : 2));
    };
    // Per-element descriptors, built once: every per-step operand is base[k*stride], so a step's
    // prologue/epilogue is a few loads and FMAs instead of index arithmetic and branches.
    //   pb  panel source P[job][slot][rhs][off_c + k]   (pc = layer slot coefficient)
    //   vb  volume source f (split or full slab) / dense test rhs
    //   tt, tbm  cell trace sources of the interfaces above / below (reconstruction pass)
    //   ob  output: Newton table rows, sampled layer row, stitched volume or dense test output
    Desc* dsm = reinterpret_cast<Desc*>(full + 3 * K1_NS + 2);  // [nel] descriptors in shared memory
    // this thread's element descriptors: registers for NC < 8 (static indices), shared memory for the
    // register-heavy DMMA path
    constexpr bool DREG = NC < 8;
    Desc dreg[DREG ? TT : 1] = {};
    auto getd = [&](int t) -> Desc {
      if constexpr (DREG) return dreg[t];
      else return dsm[tid + t * K1_CONSUMERS];
    };
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      Desc d;
      d.pb = d.vb = d.tt = d.tbm = d.ob = d.ob2 = -1;
      d.slot = 0;
      d.okind = 0;
      const int e = tid + t * K1_CONSUMERS;
      if constexpr (DREG) dreg[t] = d;
      if (e >= nel) continue;
      const int j = e / NC, q = e - (e / NC) * NC;
      const ColInfo ci = cols[q];
      if (ci.jid >= 0 && p.pass == 2) {
        d.vb = (ci.r * wzc) * w + j;
        d.ob = (ci.r * wzc) * w + j;
        d.okind = 4;
      } else if (ci.jid >= 0) {
#pragma unroll
        for (int sl = 0; sl < 4; ++sl)
          if ((ci.panmask >> sl & 1) && j == lay.prow[sl]) {
            d.pb = ((ci.jid * 4 + sl) * p.R + ci.r) * p.wx + cell.off;
            d.slot = (unsigned char)sl;
          }
        if (ci.vol == 1 && j >= lay.lo && j < lay.hi)
          d.vb = (int)(ci.r * p.f_stride) + (lay.off + j) * p.wx + cell.off;
        else if (ci.vol == 2)
          d.vb = (int)(ci.r * p.f_stride) + j * p.wx + cell.off;
        if (p.pass == 1) {
          const int tb0 = (ci.jid * p.R + ci.r) * nIc;
          if (cell.has_top) d.tt = ((tb0 + cell.cell - 1) * 2) * p.wmax + j;
          if (cell.has_bot) d.tbm = ((tb0 + cell.cell) * 2) * p.wmax + j;
          if (ci.nout < 0) {
            if (ci.vfull) {
              d.ob = (int)(ci.r * p.u_stride) + j * p.wx + cell.off;
              d.okind = 2;
            } else if (j >= lay.lo && j < lay.hi) {
              d.ob = (int)(ci.r * p.u_stride) + (lay.off + j) * p.wx + cell.off;
              d.okind = 2;
            }
          } else {
#pragma unroll
            for (int o = 0; o < 4; ++o)
              if (j == ci.opos[o]) {
                d.ob = ((ci.jid * 4 + o) * p.R + ci.r) * p.wx + cell.off;
                d.okind = 3;
              }
          }
        } else {
          d.ob = ((ci.jid * p.Lc + cell.cell) * 4 * p.R + ci.r) * p.wmax + j;
          d.okind = 1;
          if (p.s0 && ci.nout > 0) {
#pragma unroll
            for (int o = 0; o < 4; ++o)
              if (j == ci.opos[o]) d.ob2 = ((ci.jid * 4 + o) * p.R + ci.r) * p.wx + cell.off;
          }
        }
      }
      dsm[e] = d;
      if constexpr (DREG) dreg[t] = d;
    }
    // Operands of a step that do not depend on the chain are fetched ONE STEP AHEAD as raw values
    // into registers (pa: panel value, or the stored z_k / y_k of a back-substitution step;
    // pb: volume value); no arithmetic touches them until their step runs.
#define K1_FETCH(S_)                                                                                \
  do {                                                                                              \
    const int kb_ = kblk(S_);                                                                       \
    const bool back_ = kind_of(S_) == 2;                                                            \
    const bool kept_ = kb_ >= cell.lo && kb_ < cell.hi;                                             \
    const int kd_ = kind_of(S_);                                                                    \
    pcf = czero();                                                                                  \
    if (kd_ == 0) pcf = h == 0 ? p.lz[cell.lz_off + kb_] : p.uz[cell.lz_off + kb_];                 \
    else if (kd_ == 2) pcf = h == 0 ? p.uz[cell.lz_off + kb_] : p.lz[cell.lz_off + kb_];            \
    _Pragma("unroll") for (int t = 0; t < TT; ++t) {                                                \
      const int e = tid + t * K1_CONSUMERS;                                                         \
      pa[t] = czero();                                                                              \
      pb[t] = czero();                                                                              \
      if (e < nel) {                                                                                \
        if (back_) {                                                                                \
          pa[t] = Z[(size_t)kb_ * nel + e];                                                         \
        } else if (p.pass == 2) {                                                                   \
          const int vb_ = getd(t).vb;                                                               \
          if (vb_ >= 0) pb[t] = p.bd[(size_t)vb_ + (size_t)kb_ * w];                                \
        } else if (kept_) {                                                                         \
          const Desc d_ = getd(t);                                                                  \
          const int pb_ = d_.pb, vb_ = d_.vb;                                                       \
          if (pb_ >= 0) pa[t] = p.P[(size_t)pb_ + kb_];                                             \
          if (vb_ >= 0) pb[t] = p.f[(size_t)vb_ + kb_];                                             \
        }                                                                                           \
      }                                                                                             \
    }                                                                                               \
  } while (0)
    // b_k[j] from the prefetched raw operands: cell trace source + (panel + volume), the reference's
    // order of additions (sie.py:338-340)
    auto bval = [&](int k, int t, double2 va, double2 vb) -> double2 {
      const Desc d = getd(t);
      if (p.pass == 2) return vb;
      double2 inner = (d.pb >= 0 && k >= cell.lo && k < cell.hi) ? cmul(sel4(lay.coef, d.slot), va) : czero();
      inner = cadd(inner, vb);
      if (p.pass == 1) {
#pragma unroll
        for (int sl = 0; sl < 4; ++sl)
          if (k == cell.krow[sl]) {
            const int base = sl < 2 ? d.tt : d.tbm;
            if (base >= 0) inner = cadd(cmul(cell.coef[sl], p.tr[(size_t)base + (sl & 1) * p.wmax]), inner);
          }
      }
      return inner;
    };
    auto emit = [&](int k, int t, double2 x) {
      const Desc d = getd(t);
      if (d.okind == 4) {
        p.xd[(size_t)d.ob + (size_t)k * w] = x;
      } else if (d.okind >= 2) {
        if (k >= cell.lo && k < cell.hi) (d.okind == 2 ? p.u : p.smp)[(size_t)d.ob + k] = x;
      } else if (d.okind == 1) {
        if (d.ob2 >= 0 && k >= cell.lo && k < cell.hi) p.smp[(size_t)d.ob2 + k] = x;
#pragma unroll
        for (int idx = 0; idx < 4; ++idx) {
          const bool need = idx < 2 ? cell.has_top : cell.has_bot;
          if (need && k == cell.srow[idx]) p.tables[(size_t)d.ob + (size_t)idx * p.R * p.wmax] = x;
        }
      }
    };

    // optional per-phase clock64 totals of CTA 0 / thread 0 (PT_K1_TPROF)
    const bool tp = p.tprof != nullptr && blockIdx.x == 0 && tid == 0;
    long long t0 = 0, tacc[6] = {0, 0, 0, 0, 0, 0};
#define K1_TICK(I_)                           \
  do {                                        \
    if (tp) {                                 \
      const long long t_ = clock64();         \
      if ((I_) >= 0) tacc[(I_)] += t_ - t0;   \
      t0 = t_;                                \
    }                                         \
  } while (0)

    double2* cur = VA;
    double2* nxt = VB;
    int rslot = 0;      // ring slot of the next chunk
    uint32_t rph = 0;   // its fill parity
    auto ring_next = [&]() {
      if (++rslot == NS) {
        rslot = 0;
        rph ^= 1u;
      }
    };
    double2 pa[TT], pb[TT];
    double2 pcf;  // chain coefficient of the prefetched step (l_k / u_k), fetched with its operands
    K1_FETCH(0);
    // step 0 (first block of either half chain): no previous chain value
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      const int e = tid + t * K1_CONSUMERS;
      if (e < nel) cur[e] = (p.dbg & 4) ? pa[t] : bval(kblk(0), t, pa[t], pb[t]);
    }
    K1_TICK(-1);
    // Invariant at the top of step s: cur holds the matvec input of step s (formed by the previous
    // epilogue), except at the middle step, and pa/pb/pcf hold the prefetched operands of step s.
    for (int s = 0; s < nst; ++s) {
      const int kb = kblk(s);
      const int kind = kind_of(s);
      const double2 cf = pcf;
      double2 zr[TT];
      if (kind == 1) {
        const uint32_t rx = mapa(XC, (uint32_t)partner), rb = mapa(xbar, (uint32_t)partner);
        for (int e = tid; e < nel; e += K1_CONSUMERS) st_async_c(rx + (uint32_t)e * 16u, cur[e], rb);
        mbar_wait(xbar, 0);
        const double2 lm = p.lz[cell.lz_off + m], um = p.uz[cell.lz_off + m];
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const int e = tid + t * K1_CONSUMERS;
          if (e < nel) {
            const double2 zt = h == 0 ? cur[e] : XC[e];  // z_{m-1} (top chain)
            const double2 yb = h == 0 ? XC[e] : cur[e];  // y_{m+1} (bottom chain)
            cur[e] = csub(csub(bval(m, t, pa[t], pb[t]), cmul(lm, zt)), cmul(um, yb));
          }
        }
      } else if (kind == 2) {
#pragma unroll
        for (int t = 0; t < TT; ++t) zr[t] = pa[t];
      }
      K1_TICK(0);
#if K1_FETCH_POS == 0
      if (s + 1 < nst) K1_FETCH(s + 1);
#endif
      K1_TICK(1);
      named_bar(1, K1_CONSUMERS);
      K1_TICK(2);
      if constexpr (NC == 8) {
        // ---- y = Blk[kb] cur on the FP64 tensor cores: mma.sync m8n8k4 f64 (SASS DMMA.8x8x4).
        // Work items (8-row tile mt, k-step parity par) are dealt to the 7 consumer warps; per
        // k-step of 4 columns: Cr += Ar Br + (-Ai) Bi, Ci += Ar Bi + Ai Br.  A fragments come from
        // the column-major block in the ring, B fragments from cur[k][0..8).
        // K split: warp wp takes the k-steps ks = wp (mod 7) of the block and ALL NMT 8-row tiles, so
        // each warp carries 2*NMT independent accumulator chains (no per-tile predicates); the B
        // fragment of a k-step is loaded once and shared by the tiles.  Every warp arrives on every
        // chunk (count 7), having waited only for the chunks it reads.
        const int ar = lane >> 2, ak = lane & 3;
        double cm_[NMT][4];
#pragma unroll
        for (int t = 0; t < NMT; ++t) cm_[t][0] = cm_[t][1] = cm_[t][2] = cm_[t][3] = 0.0;
        for (int ch = 0; ch < nch; ++ch) {
          const int slot = rslot;
          const int ks0 = ch * (p.jc8 / 4), ks1 = min(w4, (ch + 1) * p.jc8) >> 2;
          int ks = ks0 + ((wp - ks0) % 7 + 7) % 7;  // first k-step of this warp in the chunk
          if (ks < ks1) {
            if (!(p.dbg & 1)) mbar_wait(&full[slot], rph);
            const double2* blk = reinterpret_cast<const double2*>(ring + (size_t)slot * p.slot_bytes);
            for (; ks < ks1; ks += K1_CONSUMERS / 32) {
              const int kl = (ks - ks0) * 4 + ak;  // column inside the chunk
              const double2 bv = cur[(ks * 4 + ak) * 8 + ar];
              const double2* ap = blk + kl * w + ar;
#pragma unroll
              for (int t = 0; t < NMT; ++t) {
                const double2 av = ap[t * 8];
                dmma_f64(cm_[t][0], cm_[t][1], av.x, bv.x);
                dmma_f64(cm_[t][2], cm_[t][3], av.x, bv.y);
                dmma_f64(cm_[t][0], cm_[t][1], -av.y, bv.y);
                dmma_f64(cm_[t][2], cm_[t][3], av.y, bv.x);
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_relaxed(&lempty[slot]);
          ring_next();
#if K1_FETCH_POS == 1
          // operands of the next step, issued under the matvec (used by this step's epilogue)
          if (ch == 0 && s + 1 < nst) K1_FETCH(s + 1);
#endif
        }
        K1_TICK(3);
#pragma unroll
        for (int t = 0; t < NMT; ++t) {
          const int row = t * 8 + ar;
          if (row < w) {
            red[(wp * w + row) * 8 + 2 * ak] = make_double2(cm_[t][0], cm_[t][2]);
            red[(wp * w + row) * 8 + 2 * ak + 1] = make_double2(cm_[t][1], cm_[t][3]);
          }
        }
      } else {
      // ---- y = Blk[kb] cur on the FP64 pipes.  Lane l owns rows l + 32 r (r < RW, RW = NMT here,
      // from the widest layer); warp wp owns columns wp*K1_JW .. +K1_JW of every ring chunk of
      // K1_JCD = 7*K1_JW columns.  Fixed trip counts: the loop body is K1_JW columns x RW row blocks
      // x NC right-hand sides of straight-line loads and FMAs.  Rows >= w of the last row block read
      // neighbouring shared memory and are discarded at the partial-sum write.
      constexpr int RW = NMT;
      constexpr int JW = k1_jw(NC);
      constexpr int JCD = 7 * JW;
      double2 acc[RW][NC];
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[r][q] = czero();
      for (int ch = 0; ch < nch; ++ch) {
        if (!(p.dbg & 1)) mbar_wait(&full[rslot], rph);
        const double2* blk = reinterpret_cast<const double2*>(ring + (size_t)rslot * p.slot_bytes);
        const int c0 = ch * JCD, cw = min(JCD, w - c0);
        if (!(p.dbg & 2)) {
          // all loads of the warp's JW columns first (branch-free: a column past the chunk reads
          // column 0 and multiplies a zero vector entry), then the FMAs
          double2 av[JW][RW], tv[JW][NC];
#pragma unroll
          for (int u = 0; u < JW; ++u) {
            const int jj = wp * JW + u;
            const bool ok = jj < cw;
            const int jl = ok ? jj : 0;
#pragma unroll
            for (int q = 0; q < NC; ++q) {
              const double2 t = cur[(c0 + jl) * NC + q];
              tv[u][q] = ok ? t : czero();
            }
            const double2* col = blk + jl * w + lane;
#pragma unroll
            for (int r = 0; r < RW; ++r) av[u][r] = (lane + 32 * r < w) ? col[32 * r] : czero();
          }
#pragma unroll
          for (int u = 0; u < JW; ++u)
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
              for (int q = 0; q < NC; ++q) cfma(acc[r][q], av[u][r], tv[u][q]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_relaxed(&lempty[rslot]);
        ring_next();
#if K1_FETCH_POS == 1
        // operands of the next step, issued under the matvec (used by this step's epilogue)
        if (ch == 0 && s + 1 < nst) K1_FETCH(s + 1);
#endif
      }
      K1_TICK(3);
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const int i = lane + 32 * r;
        if (i < w)
#pragma unroll
          for (int q = 0; q < NC; ++q) red[(wp * w + i) * NC + q] = acc[r][q];
      }
      }
#if K1_FETCH_POS == 2
      if (s + 1 < nst) K1_FETCH(s + 1);
#endif
      named_bar(1, K1_CONSUMERS);
      K1_TICK(4);
      // ---- epilogue: this step's output, and the matvec input of step s+1 (b_{k'} - coef * out for a
      // forward step; out itself before the middle step and for back-substitution steps)
      const int kn = s + 1 < nst ? kind_of(s + 1) : -1;
      const int kbn = s + 1 < nst ? kblk(s + 1) : 0;
      const double2 cfn = pcf;
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        const int e = tid + t * K1_CONSUMERS;
        if (e < nel) {
          const int i = e / NC, q = e - (e / NC) * NC;
          double2 y = red[i * NC + q];
          // partial sums: one set per consumer warp (DMMA k split / DFMA column split)
          static_assert(K1_CONSUMERS / 32 == 7, "partial-sum tree assumes 7 consumer warps");
          {
            const double2 p1 = red[(1 * w + i) * NC + q], p2 = red[(2 * w + i) * NC + q];
            const double2 p3 = red[(3 * w + i) * NC + q], p4 = red[(4 * w + i) * NC + q];
            const double2 p5 = red[(5 * w + i) * NC + q], p6 = red[(6 * w + i) * NC + q];
            y = cadd(cadd(cadd(y, p1), cadd(p2, p3)), cadd(cadd(p4, p5), p6));
          }
          double2 out = y;
          if (kind == 0) {
            Z[(size_t)kb * nel + e] = y;
          } else if (kind == 1) {
            if (h == 0) emit(m, t, y);
          } else {
            out = csub(zr[t], cmul(cf, y));
            if (!(p.dbg & 8)) emit(kb, t, out);
          }
          if (kn == 0) {
            const double2 b = (p.dbg & 4) ? pa[t] : bval(kbn, t, pa[t], pb[t]);
            out = csub(b, cmul(cfn, out));
          }
          nxt[e] = out;
        }
      }
      K1_TICK(5);
      double2* tmp = cur;
      cur = nxt;
      nxt = tmp;
    }
    if (tp)
      for (int i = 0; i < 6; ++i) p.tprof[i] = tacc[i];
#undef K1_FETCH
#undef K1_TICK
  }
  __syncwarp();
  cl.sync();  // no CTA leaves while a partner may still write into its shared memory
}

size_t k1_smem_bytes(int wmax, int nc, int slot_bytes, int ns) {
  // ring + three [w][NC] vectors + the [8 warps][w][NC] partial sums + column info + barriers
  return (size_t)ns * slot_bytes + (size_t)(3 * ((wmax + 3) & ~3) + k1_red_rows(wmax)) * nc * 16 +
         (size_t)nc * sizeof(ColInfo) +
         (size_t)(3 * K1_NS + 2) * 8 + (size_t)wmax * nc * sizeof(Desc) + 128;
}

cudaError_t k1_launch(const K1Params& p0, int ntasks, int nc, int wmax, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  if (nc * wmax > 4 * K1_CONSUMERS) return cudaErrorInvalidValue;  // epilogue holds <= 4 elements/thread
  if (wmax > 32 * K1_RW) return cudaErrorInvalidValue;             // w <= 128 (DFMA groups, DMMA tiles)
  static int maxsm = 0;
  if (!maxsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  // one ring slot holds one chunk (DMMA path p.jc8 columns, DFMA path 7 * k1_jw(nc)); as many slots
  // as the shared memory left next to this NC's vectors allows (<= K1_NS, a multiple of cm)
  K1Params p = p0;
  static const int jc8_env = std::getenv("PT_K1_JC8") ? atoi(std::getenv("PT_K1_JC8")) : 0;
  const long long fixed = (long long)k1_smem_bytes(wmax, nc, 0, 0);
  // DMMA path: the widest chunk (28 / 20 / 12 columns = 7 / 5 / 3 k-steps) that still leaves >= 4 ring slots;
  // 7 k-steps per chunk give every consumer warp one k-step of each chunk (cfg2: 9.9 -> 9.8 ms per step)
  p.jc8 = K1_JC8;
  if (jc8_env >= 4) {
    p.jc8 = jc8_env & ~3;
  } else {
    for (int cand : {28, 20, 12}) {
      const long long sl = (16LL * wmax * cand + 127) / 128 * 128;
      if (((long long)maxsm - fixed) / sl >= 4) {
        p.jc8 = cand;
        break;
      }
    }
  }
  const int jc = nc == 8 ? p.jc8 : 7 * k1_jw(nc);
  const long long slot = (16LL * wmax * jc + 127) / 128 * 128;
  int ns = (int)std::min<long long>(K1_NS, ((long long)maxsm - fixed) / slot);
  ns -= ns % p.cm;
  if (ns < 2) return cudaErrorInvalidValue;
  p.slot_bytes = (int)slot;
  p.ns = ns;
  const size_t smax = k1_smem_bytes(wmax, nc, p.slot_bytes, ns);
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
#define PT_K1_GO(N, M)                                                                                \
  {                                                                                                   \
    set_smem_attr((const void*)k1_twisted<N, M>, smax);                                              \
    if (2 * p.cm > 8) cudaFuncSetAttribute(k1_twisted<N, M>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); \
    return cudaLaunchKernelEx(&cfg, k1_twisted<N, M>, p);                                             \
  }
  if (nc == 8) {
    switch ((wmax + 7) >> 3) {  // 8-row tiles of the widest layer (DMMA path)
      case 1: case 2: case 3: case 4: case 5: case 6: case 7: case 8: PT_K1_GO(8, 8)
      case 9: PT_K1_GO(8, 9)
      case 10: PT_K1_GO(8, 10)
      case 11: PT_K1_GO(8, 11)
      case 12: PT_K1_GO(8, 12)
      case 13: case 14: PT_K1_GO(8, 14)
      case 15: case 16: PT_K1_GO(8, 16)
      default: return cudaErrorInvalidValue;
    }
  }
  const int rw = (wmax + 31) >> 5;  // DFMA path: row blocks of 32 lanes
#define PT_K1_RW(N)                        \
  switch (rw) {                            \
    case 1: PT_K1_GO(N, 1)                 \
    case 2: PT_K1_GO(N, 2)                 \
    case 3: PT_K1_GO(N, 3)                 \
    case 4: PT_K1_GO(N, 4)                 \
    default: return cudaErrorInvalidValue; \
  }
  switch (nc) {
    case 1: PT_K1_RW(1)
    case 2: PT_K1_RW(2)
    case 4: PT_K1_RW(4)
    default: return cudaErrorInvalidValue;
  }
#undef PT_K1_RW
#undef PT_K1_GO
}
