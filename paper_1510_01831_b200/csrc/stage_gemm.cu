// Many-RHS form of the two dense products of a sample-only layer solve (the tensor-core regime of the north
// star: >= 32 columns per product):
//
//   pass-0 product      out[m][n] = sum_{s,k} Q0[m][(s,k)] P[job(n)][s][q(n)][off_c + lo + k]
//                       (the first cell-solve pass of LayerOperator.boundary_samples, subdomain.py:184-199, with
//                       the offline pass-0 operators; rows = Newton-table rows then layer-row samples), and
//   sampled response    smp[(k,o)][r] += sum_{s,j} gsmp[k][o][s][j] tr_s[r][j]
//                       (the reconstruction pass of the same layer solve sampled at the layer trace rows,
//                       nested.py:344-353 by linearity),
//
// as one streaming complex GEMM kernel: C[M x N] = A[M x K] B[K x N] per (job or layer group, cell), A the
// offline operator (row-major, K contiguous), B the gathered panels (column-major, K contiguous).  The small-N
// kernels (k_pass0, k_green_samples2: one 8-row tile x 16 columns per warp group, operands straight from L2)
// stay for fewer columns.
//
// CTA = 8 consumer warps + 1 producer warp, one CTA per SM, persistent over (problem, row block, column block)
// work items.  A CTA tile is MT x NT = 4 x 8 (32 rows x 64 columns) or 8 x 4 eight-wide tiles; K streams in
// chunks of 64 (2-slot ring) or 32 (4 slots) through shared memory: the producer warp issues one cp.async.bulk per operator row
// and per panel column of the chunk (<= 96 copies of 1 KB / 512 B, completion on the slot.s mbarrier), rows padded by
// 4 double2 so the DMMA fragment loads (LDS.128, row = lane / 4, k = lane % 4) are conflict-free.  Every
// consumer warp owns a 2 x 2 block of (row tile, column tile) pairs over the whole K: four independent
// accumulator chains per pair (Ar Br, Ai Bi, Ar Bi, Ai Br), 16 DMMAs per 4 fragment loads, no cross-warp
// reduction; the sum over K runs in a fixed order (deterministic).  Epilogues as in stage_dev.cuh.
#include <cstdlib>

#include "pt_launch.cuh"
#include "stage_dev.cuh"

#define SG_T 256
#define SG_TB (SG_T + 32)
#define SG_RC 96
// K rows per chunk (template parameter KC): 32 with a 4-slot ring or 64 with a 2-slot ring (copies twice as
// long: half the bulk-copy requests per flop); rows padded by 4 double2 (row stride = 4 mod 8 sixteen-byte
// units: conflict-free LDS.128 fragment loads)
#define SG_LD (KC + 4)
#define SG_NSLOT (KC == 32 ? 4 : 2)
#define SG_SLOT (SG_RC * SG_LD)  // double2 per ring slot
#define SG_KC KC

struct SgArgs {
  const OJob* jobs;
  const CellInfo* cells;
  const LayerInfo* layers;
  int R, Lc, wx, wmax, nprob, rbmax, cbmax;
  double2* smp;
  // sampled response
  const double2* gsmp;
  const double2* tr;
  int fuse_combine;
  VecTab tab;
  const int* rmap;
  // pass-0 product
  const int* grp;
  const int* ljobs;
  const double2* q0;
  const double2* P;
  double2* tables;
  int accum;
  RhsOut ro;
};

struct SgDesc {
  int M, N, m0, n0;
  int nseg, segs, klen;
  int jid, c, layer, nout, jb0, nj, lo, off, w;
  long long aseg, abase, bbase;
  long long bslot;  // B offset per slot unit (MODE 1: s * bslot; MODE 0: ((s < 2 ? c - 1 : c) * 2 + (s & 1)) * bslot)
  long long arow;   // A row stride (elements)
};

template <int MODE>
__device__ __forceinline__ long long sg_boff(const SgDesc& d, int s) {
  return MODE == 0 ? (long long)((s < 2 ? d.c - 1 : d.c) * 2 + (s & 1)) * d.bslot : (long long)s * d.bslot;
}

// (problem, row block, column block) of work item `it`; false: nothing to do (warp-uniform)
template <int MODE, int MT, int NT>
__device__ __forceinline__ bool sg_desc(const SgArgs& a, int it, SgDesc& d) {
  const int per = a.rbmax * a.cbmax;
  const int prob = it / per, rem = it - prob * per;
  const int rb = rem / a.cbmax, cb = rem - rb * a.cbmax;
  d.m0 = rb * MT * 8;
  d.n0 = cb * NT * 8;
  d.c = prob % a.Lc;
  const int g = prob / a.Lc;
  if (MODE == 0) {  // sampled response: problem = (job, cell)
    d.jid = g;
    const OJob& jb = a.jobs[g];
    d.nout = jb.nout;
    if (d.nout <= 0) return false;
    d.layer = jb.layer;
    const CellInfo& ci = a.cells[d.layer * a.Lc + d.c];
    d.w = ci.w;
    d.lo = ci.lo;
    d.off = ci.off;
    d.M = (ci.hi - ci.lo) * d.nout;
    d.N = a.R;
    const int s_lo = ci.has_top ? 0 : 2, s_hi = ci.has_bot ? 4 : 2;
    d.nseg = s_hi - s_lo;
    d.segs = 0;
    for (int s = s_lo, i = 0; s < s_hi; ++s, ++i) d.segs |= s << (2 * i);
    d.klen = ci.w;
    d.aseg = ci.w;
    d.abase = ci.gsmp_off;
    d.arow = 4LL * ci.w;
    const int nIc = a.Lc - 1;
    d.bbase = (long long)g * a.R * nIc * 2 * a.wmax;
    d.bslot = a.wmax;
  } else {  // pass-0 product: problem = (layer group, cell)
    d.layer = a.grp[3 * g];
    d.jb0 = a.grp[3 * g + 1];
    d.nj = a.grp[3 * g + 2];
    const CellInfo& ci = a.cells[d.layer * a.Lc + d.c];
    d.w = ci.w;
    d.lo = ci.lo;
    d.off = ci.off;
    const int nk = ci.hi - ci.lo, nk4 = (nk + 3) & ~3;
    d.M = q0_rows(ci.w, nk);  // device row layout (pt_device.cuh): table rows, then the sample rows by output row
    d.N = d.nj * a.R;
    if (d.m0 >= d.M || d.n0 >= d.N) return false;
    const int tab8 = q0_tab8(ci.w), nk8 = q0_nk8(nk);
    if (d.m0 >= tab8) {  // a block of sample rows: skipped when no job of these columns samples its output rows
      const int o0 = (d.m0 - tab8) / nk8, o1 = (min(d.m0 + MT * 8, d.M) - 1 - tab8) / nk8;
      const int ln = a.layers[d.layer].n;
      bool need = false;
      for (int jj = d.n0 / a.R; jj < d.nj && jj * a.R < d.n0 + NT * 8; ++jj) {
        const OJob& jo = a.jobs[a.ljobs[d.jb0 + jj]];
        for (int o = 0; o < jo.nout; ++o) {
          const int orow = jo.orow[o];
          const int oi = orow == 0 ? 0 : (orow == 1 ? 1 : (orow == ln ? 2 : 3));
          need |= oi >= o0 && oi <= o1;
        }
      }
      if (!need) return false;
    }
    int used = 0;
    for (int jj = 0; jj < d.nj; ++jj) {
      const OJob& jo = a.jobs[a.ljobs[d.jb0 + jj]];
#pragma unroll
      for (int s = 0; s < 4; ++s) used |= (jo.pan[s][0].vec >= 0) << s;
    }
    d.nseg = 0;
    d.segs = 0;
    for (int s = 0; s < 4; ++s)
      if (used >> s & 1) d.segs |= s << (2 * d.nseg++);
    d.klen = nk;
    d.aseg = nk4;
    d.abase = ci.q0_off;
    d.arow = 4LL * nk4;
    d.bbase = ci.off + ci.lo;
    d.bslot = (long long)a.R * a.wx;
  }
  return d.m0 < d.M && d.n0 < d.N && d.nseg > 0;
}

__device__ __forceinline__ void sg_dmma4(double (&q)[8], double ar, double ai, double br, double bi) {
  dmma_f64(q[0], q[1], ar, br);
  dmma_f64(q[2], q[3], ai, bi);
  dmma_f64(q[4], q[5], ar, bi);
  dmma_f64(q[6], q[7], ai, br);
}

template <int MODE, int MT, int NT, int KC>
__global__ void __launch_bounds__(SG_TB, 1) k_stage_gemm(const SgArgs a, int nitems) {
  extern __shared__ __align__(128) unsigned char sg_smem[];
  double2* ring = reinterpret_cast<double2*>(sg_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(sg_smem + sizeof(double2) * SG_NSLOT * SG_SLOT);
  uint64_t* empty = full + SG_NSLOT;
  const int tid = threadIdx.x, wp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < SG_NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], SG_T / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const double2* Aop = MODE == 0 ? a.gsmp : a.q0;
  const double2* Bop = MODE == 0 ? a.tr : a.P;
  if (wp == 8) {
    // ---- producer: the chunks of this CTA's work items in the consumers' order
    int issued = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      SgDesc d;
      if (!sg_desc<MODE, MT, NT>(a, it, d)) continue;
      const int mvalid = min(MT * 8, d.M - d.m0), nvalid = min(NT * 8, d.N - d.n0);
      // this lane's three (row | column) sources, slot-independent part
      const double2* src[3];
      int dstrow[3];
      bool isA[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int idx = lane + 32 * i;
        dstrow[i] = idx;
        src[i] = nullptr;
        isA[i] = idx < MT * 8;
        if (isA[i]) {
          if (idx < mvalid) {
            const int m = d.m0 + idx;
            if (MODE == 0) {
              const int mk = m / d.nout, mo = m - mk * d.nout;
              const int orow = a.jobs[d.jid].orow[mo];
              const int oi = orow == 0 ? 0 : (orow == 1 ? 1 : (orow == a.layers[d.layer].n ? 2 : 3));
              src[i] = Aop + d.abase + ((long long)(d.lo + mk) * 4 + oi) * d.arow;
            } else {
              src[i] = Aop + d.abase + (long long)m * d.arow;
            }
          }
        } else {
          const int nn = idx - MT * 8;
          if (nn < nvalid) {
            const int n = d.n0 + nn;
            if (MODE == 0) {
              src[i] = Bop + d.bbase + (long long)n * (a.Lc - 1) * 2 * a.wmax;
            } else {
              const int jid = a.ljobs[d.jb0 + n / a.R], q = n % a.R;
              src[i] = Bop + ((long long)jid * 4 * a.R + q) * a.wx + d.bbase;
            }
          }
        }
      }
      for (int si = 0; si < d.nseg; ++si) {
        const int s = d.segs >> (2 * si) & 3;
        for (int k0 = 0; k0 < d.klen; k0 += SG_KC, ++issued) {
          const int slot = issued % SG_NSLOT;
          if (issued >= SG_NSLOT) {
            if (lane == 0) mbar_wait_suspend(&empty[slot], ((issued / SG_NSLOT) - 1) & 1u);
            __syncwarp();
          }
          const int kv = min(SG_KC, d.klen - k0);
          const uint32_t bytes = (uint32_t)kv * 16u;
          if (lane == 0) mbar_expect_tx_relaxed(&full[slot], bytes * (uint32_t)(mvalid + nvalid));
          __syncwarp();
          double2* sp = ring + (size_t)slot * SG_SLOT;
#pragma unroll
          for (int i = 0; i < 3; ++i)
            if (src[i])
              bulk_g2s(sp + (size_t)dstrow[i] * SG_LD, src[i] + (isA[i] ? (long long)s * d.aseg : sg_boff<MODE>(d, s)) + k0, bytes,
                       &full[slot]);
        }
      }
    }
    return;
  }
  // ---- consumers
  constexpr int WMN = MT / 2;  // warp blocks along M
  const int wmi = wp % WMN, wni = wp / WMN;
  const int r8 = lane >> 2, kl = lane & 3;
  int done = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    SgDesc d;
    if (!sg_desc<MODE, MT, NT>(a, it, d)) continue;
    double acc[2][2][8];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[x][y][e] = 0.0;
    // warp-uniform: this warp's block holds at least one valid (row tile, column tile) pair
    const bool wact = d.m0 + wmi * 16 < d.M && d.n0 + wni * 16 < d.N;
    for (int si = 0; si < d.nseg; ++si)
      for (int k0 = 0; k0 < d.klen; k0 += SG_KC, ++done) {
        const int slot = done % SG_NSLOT;
        mbar_wait_suspend(&full[slot], (done / SG_NSLOT) & 1u);
        const int kv = min(SG_KC, d.klen - k0);
        if (wact) {
          const double2* A0 = ring + (size_t)slot * SG_SLOT + (size_t)(wmi * 16 + r8) * SG_LD + kl;
          const double2* B0 = ring + (size_t)slot * SG_SLOT + (size_t)(MT * 8 + wni * 16 + r8) * SG_LD + kl;
          const int nkf = kv >> 2;
#pragma unroll 4
          for (int ks = 0; ks < nkf; ++ks) {
            const double2 a0 = A0[ks * 4], a1 = A0[8 * SG_LD + ks * 4], b0 = B0[ks * 4], b1 = B0[8 * SG_LD + ks * 4];
            sg_dmma4(acc[0][0], a0.x, a0.y, b0.x, b0.y);
            sg_dmma4(acc[0][1], a0.x, a0.y, b1.x, b1.y);
            sg_dmma4(acc[1][0], a1.x, a1.y, b0.x, b0.y);
            sg_dmma4(acc[1][1], a1.x, a1.y, b1.x, b1.y);
          }
          if (kv & 3) {  // the chunk's last, partial k-step: rows of the ring beyond kv hold stale data
            const bool kin = kl < (kv & 3);
            double2 a0 = czero(), a1 = czero(), b0 = czero(), b1 = czero();
            if (kin) {
              a0 = A0[nkf * 4];
              a1 = A0[8 * SG_LD + nkf * 4];
              b0 = B0[nkf * 4];
              b1 = B0[8 * SG_LD + nkf * 4];
            }
            sg_dmma4(acc[0][0], a0.x, a0.y, b0.x, b0.y);
            sg_dmma4(acc[0][1], a0.x, a0.y, b1.x, b1.y);
            sg_dmma4(acc[1][0], a1.x, a1.y, b0.x, b0.y);
            sg_dmma4(acc[1][1], a1.x, a1.y, b1.x, b1.y);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_relaxed(&empty[slot]);
      }
    if (!wact) continue;
    // ---- epilogue: C fragment = row r8 of the tile, columns 2 kl and 2 kl + 1
    const CellInfo& ci = a.cells[d.layer * a.Lc + d.c];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int m = d.m0 + (wmi * 2 + x) * 8 + r8;
      if (m >= d.M) continue;
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = d.n0 + (wni * 2 + y) * 8 + 2 * kl + h;
          if (n >= d.N) continue;
          const double* q = acc[x][y];
          const double2 v = make_double2(q[h] - q[2 + h], q[4 + h] + q[6 + h]);
          if (MODE == 0) {
            const OJob& jb = a.jobs[d.jid];
            const int mk = m / d.nout, mo = m - mk * d.nout;
            const int xg = ci.off + ci.lo + mk;
            double2* dst = a.smp + ((size_t)(d.jid * 4 + mo) * a.R + n) * a.wx + xg;
            const double2 yv = cadd(*dst, v);
            if (!a.fuse_combine) {
              *dst = yv;
            } else {  // out = scoef*sample + add - (sub0 + sub1) (k_combine)
              const int r = a.rmap[n];
              double2 o = cscale(yv, jb.scoef[mo]);
              if (jb.add[mo].vec >= 0) o = cadd(o, vref(a.tab, jb.add[mo], r, xg, a.wx));
              if (jb.sub[mo][0].vec >= 0) {
                double2 sb = vref(a.tab, jb.sub[mo][0], r, xg, a.wx);
                if (jb.sub[mo][1].vec >= 0) sb = cadd(sb, vref(a.tab, jb.sub[mo][1], r, xg, a.wx));
                o = csub(o, sb);
              }
              const VecView& dv = a.tab.v[jb.dst[mo].vec];
              dv.p[(size_t)r * dv.stride + (size_t)jb.dst[mo].seg * a.wx + xg] = o;
            }
          } else {
            const int w = ci.w, nk = ci.hi - ci.lo, tab8 = q0_tab8(w), nk8 = q0_nk8(nk);
            if (m >= 4 * w && (m < tab8 || (m - tab8) % nk8 >= nk)) continue;  // padding rows
            const int jid = a.ljobs[d.jb0 + n / a.R], qq = n % a.R;
            if (m < 4 * w) {
              const int idx = m / w, j = m - idx * w;
              double2* tp = a.tables + ((((size_t)jid * a.Lc + d.c) * 4 + idx) * a.R + qq) * a.wmax + j;
              const double2 tv = a.accum ? cadd(*tp, v) : v;
              *tp = tv;
              if (a.ro.base) {  // rows n, n+1 of cell c < nI feed down[c]; rows 0, 1 of cell c >= 1 feed up[c - 1]
                const int nIc = a.Lc - 1;
                int seg = -1;
                if (idx >= 2 && d.c < nIc) seg = 2 * d.c + (idx - 2);
                else if (idx < 2 && d.c >= 1) seg = 2 * nIc + 2 * (d.c - 1) + idx;
                if (seg >= 0)
                  a.ro.base[((size_t)jid * a.R + qq) * a.ro.stride + a.ro.off + (size_t)seg * w + j] =
                      make_double2(-tv.x, -tv.y);
              }
            } else {
              const int mm = m - tab8, oi = mm / nk8, kk = mm - oi * nk8;
              const OJob& jb = a.jobs[jid];
              const int ln = a.layers[d.layer].n;
              for (int o = 0; o < jb.nout; ++o) {
                const int orow = jb.orow[o];
                const int ok_ = orow == 0 ? 0 : (orow == 1 ? 1 : (orow == ln ? 2 : 3));
                if (ok_ == oi) a.smp[((size_t)(jid * 4 + o) * a.R + qq) * a.wx + ci.off + ci.lo + kk] = v;
              }
            }
          }
        }
    }
  }
}

template <int KC>
constexpr size_t sg_smem() {
  return sizeof(double2) * SG_NSLOT * SG_SLOT + 2 * SG_NSLOT * sizeof(uint64_t);
}
static_assert(sg_smem<32>() <= 232448 && sg_smem<64>() <= 232448, "k_stage_gemm exceeds 227 KB of shared memory");

// columns per product from which the streaming GEMM replaces the small-N kernels: the sampled response from 1
// (measured faster at every column count: cfg5 1 RHS 73 -> 51 ms per solve, 8 RHS 77 -> 58 ms; cfg3 1 RHS 11.2 ->
// 9.7 ms), the pass-0 product from 32 (below, k_pass0's many small CTAs stream the operator faster: cfg5 1 RHS
// 90 against 98 ms).  PT_SGEMM_MIN sets both; PT_NO_SGEMM keeps the small-N kernels everywhere.
int stage_gemm_min_cols(int mode) {
  static int v[2] = {-1, -1};
  if (v[0] < 0) {
    v[0] = 1;
    v[1] = 32;
    if (const char* e = std::getenv("PT_SGEMM_MIN")) v[0] = v[1] = std::max(1, atoi(e));
    if (std::getenv("PT_NO_SGEMM")) v[0] = v[1] = 1 << 30;
  }
  return v[mode ? 1 : 0];
}

template <int MODE>
static cudaError_t sg_launch(const SgArgs& a0, int M_max, int N_max, int num_sms, cudaStream_t st) {
  SgArgs a = a0;
  // 4 x 8 tiles (32 rows x 64 columns: the operator is streamed once) unless 8 x 4 pads the columns less
  const bool wide = (N_max + 63) / 64 * 64 <= (N_max + 31) / 32 * 32;
  const int mt = wide ? 4 : 8, nt = wide ? 8 : 4;
  a.rbmax = (M_max + mt * 8 - 1) / (mt * 8);
  a.cbmax = (N_max + nt * 8 - 1) / (nt * 8);
  const long long nitems = (long long)a.nprob * a.rbmax * a.cbmax;
  if (nitems <= 0) return cudaSuccess;
  if (nitems > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = (int)std::min<long long>(nitems, num_sms);
  static const int kc = std::getenv("PT_SG_KC") ? atoi(std::getenv("PT_SG_KC")) : 64;
#define SG_GO(MT_, NT_, KC_)                                                             \
  {                                                                                      \
    set_smem_attr((const void*)k_stage_gemm<MODE, MT_, NT_, KC_>, sg_smem<KC_>());       \
    k_stage_gemm<MODE, MT_, NT_, KC_><<<grid, SG_TB, sg_smem<KC_>(), st>>>(a, (int)nitems); \
  }
  if (wide) {
    if (kc == 32) SG_GO(4, 8, 32) else SG_GO(4, 8, 64)
  } else {
    if (kc == 32) SG_GO(8, 4, 32) else SG_GO(8, 4, 64)
  }
#undef SG_GO
  return cudaGetLastError();
}

cudaError_t sample_gemm_launch(const OJob* jobs, int J, const CellInfo* cells, const LayerInfo* layers,
                               const double2* gsmp, const double2* tr, double2* smp, int R, int Lc, int wx, int wmax,
                               int kmax, int num_sms, cudaStream_t st, const VecTab* tab, const int* rmap) {
  SgArgs a{};
  a.jobs = jobs;
  a.cells = cells;
  a.layers = layers;
  a.R = R;
  a.Lc = Lc;
  a.wx = wx;
  a.wmax = wmax;
  a.nprob = J * Lc;
  a.smp = smp;
  a.gsmp = gsmp;
  a.tr = tr;
  a.fuse_combine = tab != nullptr;
  if (tab) a.tab = *tab;
  a.rmap = rmap;
  return sg_launch<0>(a, kmax * 4, R, num_sms, st);
}

cudaError_t pass0_gemm_launch(const int* grp, int ngroups, const int* ljobs, const OJob* jobs, const CellInfo* cells,
                              const LayerInfo* layers, const double2* q0, const double2* P, double2* tables,
                              double2* smp, int R, int Lc, int wx, int wmax, int kmax, int max_jobs_per_layer,
                              int num_sms, cudaStream_t st, int accum, const RhsOut* rhs_out) {
  SgArgs a{};
  a.jobs = jobs;
  a.cells = cells;
  a.layers = layers;
  a.R = R;
  a.Lc = Lc;
  a.wx = wx;
  a.wmax = wmax;
  a.nprob = ngroups * Lc;
  a.smp = smp;
  a.grp = grp;
  a.ljobs = ljobs;
  a.q0 = q0;
  a.P = P;
  a.tables = tables;
  a.accum = accum;
  a.ro = rhs_out ? *rhs_out : RhsOut{nullptr, 0, 0};
  return sg_launch<1>(a, q0_rows(wmax, kmax), max_jobs_per_layer * R, num_sms, st);
}
