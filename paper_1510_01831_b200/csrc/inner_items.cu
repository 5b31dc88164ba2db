// Inner polarized-traces GMRES over the Green-block item programs, whole GPU, all right-hand sides of a job
// per tensor-core tile (replaces _InnerPT.solve_traces, nested.py:134-153, for layers whose dense inner
// operators are not built: Lc > 8).
//
// Every instance (layer-solve job, RHS) runs exactly the Krylov process of krylov.gmres (krylov.py:53-135):
// b = pre(rhs), beta0 = ||b||, V_0 = b / beta0, then w = pre(op(V_j)), Arnoldi, complex Givens, stop when
// |g_{j+1}| / beta0 <= inner_ktol, x = V_k y.  The operator (inner apply_M_polarized, sie.py:203-228) and the
// preconditioner (inner precondition_gs, sie.py:272-326) are the host-built item programs (solver.cu
// build_inner): one item is one sampled panel  sum_slot G[cell][row][slot] @ panel_slot + add - sub, which is
// CellBlockLayer.boundary_samples (nested.py:113-122) plus the reference's elementwise steps.
//
// Layout.  Inner vectors are RHS-minor: per job [vector][n-tile][element][8 instances] (double2), so the
// panel of one vector segment for 8 RHS is one contiguous [w][8] block, exactly the shape of a Green tile
// ([w][8 rows], tile-major, k_green_tiles).  A program phase is a set of independent (job, item) GEMMs
// C[w x R] = sum_slot G_slot[w x w] B_slot[w x R]; they are cut into CTA tiles of MTC row tiles x NTC n-tiles
// (the config per phase is chosen so the tiles fill the GPU), the K dimension (slot, k) streams through a
// shared-memory ring in 32-row chunks by cp.async.bulk (one copy per row tile / n-tile and chunk, completion
// on an mbarrier), and the products run on the FP64 tensor cores (mma.sync m8n8k4, SASS DMMA): each warp owns
// WM x WN (row tile, n-tile) pairs over a part of K with four independent accumulator chains per pair
// (Ar Br, Ai Bi, Ar Bi, Ai Br).  Partial tiles are summed in shared memory in a fixed order (deterministic).
// Phases are separated by grid barriers (cooperative launch, one CTA per SM).
//
// Arnoldi.  The orthogonalisation is classical Gram-Schmidt with one reorthogonalisation (CGS2), split over
// the whole GPU by (job, n-tile, element slice): the projections h = V^T w are reduced once per pass from
// per-slice partials in a fixed order, so every CTA sees the same bits.  In exact arithmetic CGS2 and the
// reference's MGS give the same Hessenberg column; both keep the basis orthonormal to working precision for
// these short Krylov runs, so the iterate x_k and the per-instance iteration counts are the reference's
// ("MGS vs CGS2 is harmless: x_k is the same minimiser over the same Krylov space").  Three passes
// and grid barriers per step: h1 = V^H w; w' = w - V h1 with h2 = V^H w' and ||w'||^2; then V_{j+1} = (w' - V h2) / hn
// with hn^2 = ||w'||^2 - ||h2||^2 (w'' is orthogonal to V to rounding, so its norm is known before it is formed
// and the vector is stored normalised without a fourth pass).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "pt_launch.cuh"

namespace cg = cooperative_groups;

#define II_T 256           // consumer threads per CTA (8 warps)
#define II_TB (II_T + 32)  // + one producer warp (warp 8) that only issues the ring's bulk copies
#define II_RING (144 * 1024)
#define II_NSLOT 16
#define II_RED (32 * 1024)
#define II_MAXJ 64
#define II_MAXNT 32
#define II_SMAX 16     // element slices per (job, n-tile) in the vector phases
#define II_MAXIT 320   // op + pre program items (staged in shared memory, compact form)
#define II_MAXPH 256   // program phases
#define II_JREG 4      // Arnoldi steps whose basis entries stay in registers (beyond: a slower loop)

struct TileCfg {
  int mtc, ntc, wm, wn, kw;
};
// CTA tile shapes: MTC row tiles x NTC n-tiles; warps = (MTC/WM) x (NTC/WN) x KW = 8.  2 x 2 warp blocks
// wherever the tile allows (a warp product with one A and one B fragment per 4 DMMAs reaches only about half
// of the DMMA rate: shared-memory fragment loads and DMMAs share the issue path; tools/chunk_mma_micro.cu).
#define II_NCFG 7
__device__ __constant__ TileCfg II_CFG[II_NCFG] = {{8, 4, 2, 2, 1}, {4, 4, 2, 2, 2}, {4, 2, 2, 2, 4}, {2, 2, 2, 2, 8},
                                                   {4, 1, 2, 1, 4}, {2, 1, 2, 1, 8}, {1, 1, 1, 1, 8}};
// relative DMMA issue rate of a warp block (measured: 2x2 0.23, 2x1 0.165, 1x1 0.12 DMMA/clk/SM)
__device__ __forceinline__ float cfg_rate(const TileCfg& c) {
  return c.wm * c.wn == 4 ? 0.23f : (c.wm * c.wn == 2 ? 0.165f : 0.12f);
}

// optional clock64 segment totals of CTA 0 (PT_INNER_TPROF): 0 phase setup, 1 chunk loop, 2 epilogue,
// 3 program-phase grid barriers, 4 vector passes, 5 vector grid barriers, 6 init, 7 final, 8 phases, 9 tiles
__device__ unsigned long long g_ii_t[16];
__device__ unsigned long long g_ii_w[1024];  // per CTA: cycles outside grid barriers (PT_INNER_TPROF)
__device__ unsigned long long g_ii_tiles[1024];  // per CTA: tiles processed (PT_INNER_TPROF)
// event trace of one CTA's thread 0 (PT_II_TRACE=<cta+1>): (code << 48 | arg << 32 | clock low bits)
#define II_NEV 4096
__device__ unsigned long long g_ii_ev[II_NEV];
struct IITrace {
  bool on;
  int n;
  __device__ void ev(int code, int arg) {
    if (on && n < II_NEV)
      g_ii_ev[n++] = ((unsigned long long)code << 56) | ((unsigned long long)(arg & 0xffffff) << 32) |
                     (unsigned long long)(unsigned)clock64();
  }
};
struct IITick {  // fire-and-forget atomics: the timed thread never waits on the counters
  bool on;
  long long t0;
  __device__ void start() {
    if (on) t0 = clock64();
  }
  __device__ void tick(int i) {
    if (on) {
      const long long t = clock64();
      atomicAdd(&g_ii_t[i], (unsigned long long)(t - t0));
      t0 = t;
    }
  }
  __device__ void count(int i) {
    if (on) atomicAdd(&g_ii_t[i], 1ULL);
  }
};

// program item as staged in shared memory: IItem with 16-bit references (vector id, segment)
struct RefS {
  short vec, seg;
};
struct IItemS {
  short cell, row;
  RefS pan[4][2];
  RefS dst, add[2], sub[2], rev;
  int flags;
};
__device__ __forceinline__ RefS refs(const Ref& r) { return RefS{(short)r.vec, (short)r.seg}; }
__device__ __forceinline__ IItemS pack_item(const IItem& it) {
  IItemS o;
  o.cell = (short)it.cell;
  o.row = (short)it.row;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    o.pan[s][0] = refs(it.pan[s][0]);
    o.pan[s][1] = refs(it.pan[s][1]);
  }
  o.dst = refs(it.dst);
  o.add[0] = refs(it.add[0]);
  o.add[1] = refs(it.add[1]);
  o.sub[0] = refs(it.sub[0]);
  o.sub[1] = refs(it.sub[1]);
  o.rev = refs(it.rev);
  o.flags = it.flags;
  return o;
}

struct IIShared {
  uint64_t full[II_NSLOT];
  uint64_t empty[II_NSLOT];  // one arrive per consumer warp
  double dred[2 * II_T / 32 * 8];
  int nact[II_MAXJ];                        // active n-tiles per job
  unsigned char act[II_MAXJ][II_MAXNT];     // active n-tile ids per job
  unsigned char amask[II_MAXJ][II_MAXNT];   // active instance bitmask per (job, n-tile)
  int jw[II_MAXJ], jlay[II_MAXJ], jjob[II_MAXJ];
  int tpre[II_NCFG][II_MAXJ + 1];           // per config: prefix over jobs of CTA tiles per item
  unsigned char ins[II_MAXIT];              // slot count of every program item
  IItemS items[II_MAXIT];                   // the op + pre programs (staged once)
  // vector-phase staging (aliases the program phases' reduction buffer): per instance of a (job, n-tile)
  double2 (*gv)[3][34];                     // Givens: column, cs, sn / back substitution: g and triangle
  double2 (*yv)[34];                        // x = V y coefficients, [33] = k
  int phw[II_MAXPH];                        // per program phase (op phases first): sum of item weights
  unsigned char phcfg[II_MAXPH];            // per program phase: tile shape for the current active sets
  unsigned char phtwo[II_MAXPH];            // per program phase: some item has a two-term panel
  int any_active;
};

__device__ __forceinline__ double2* v2p(const InnerParams& p, int job, int v, int nt) {
  return p.scratch + (size_t)job * p.s2_job + (size_t)v * p.s2_vec + (size_t)nt * p.nmax * 8;
}

// per-item partials of the vector phases: [area][vector work item][m][8] double2
__device__ __forceinline__ double2* partp(const InnerParams& p, int area, int v) {
  const size_t rec = (size_t)(p.cap + 2) * 8;
  return p.part + ((size_t)area * p.part_items + v) * rec;
}

// barrier of the 8 consumer warps only (the producer warp never waits on the consumers' shared-memory work)
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ void dmma4(double (&a)[8], double ar, double ai, double br, double bi) {
  dmma_f64(a[0], a[1], ar, br);
  dmma_f64(a[2], a[3], ai, bi);
  dmma_f64(a[4], a[5], ar, bi);
  dmma_f64(a[6], a[7], ai, br);
}

// ---------------------------------------------------------------------------------------- tile enumeration
// The CTA tiles of one phase are numbered item-major, then job, then row-tile group, then n-tile group, and dealt
// round-robin to the CTAs (tile t -> CTA t mod G): every CTA gets a near-equal share of every item's tiles.
// Decoding a number is a few 32-bit divisions and a binary search over the per-job prefix (no serial search
// over the phase, no 64-bit division on the critical path after the grid barrier).
__device__ __forceinline__ int item_ns_g(const IItem& it) {
  int ns = 0;
  if (it.cell >= 0)
    for (int s = 0; s < 4; ++s) ns += it.pan[s][0].vec >= 0;
  return ns;
}

struct Geo {
  int nmtg, nntg;
};
__device__ __forceinline__ Geo job_geo(const IIShared& S, const TileCfg& c, int jx) {
  const int nmt = (S.jw[jx] + 7) >> 3;
  return Geo{(nmt + c.mtc - 1) / c.mtc, (S.nact[jx] + c.ntc - 1) / c.ntc};
}

struct TileRef {
  int jx, ii, mtg, ntg;  // job, item (phase-local), row-tile group, n-tile group
};
__device__ __forceinline__ TileRef tile_decode(const IIShared& S, int cfg, int J, int t) {
  const int tpi = S.tpre[cfg][J];
  TileRef r;
  r.ii = t / tpi;
  int rem = t - r.ii * tpi;
  int lo = 0, hi = J - 1;  // last job whose prefix <= rem
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (S.tpre[cfg][mid] <= rem) lo = mid;
    else hi = mid - 1;
  }
  r.jx = lo;
  rem -= S.tpre[cfg][lo];
  const int nntg = (S.nact[lo] + II_CFG[cfg].ntc - 1) / II_CFG[cfg].ntc;
  r.mtg = rem / nntg;
  r.ntg = rem - r.mtg * nntg;
  return r;
}

// ---------------------------------------------------------------------------------------- tiles and chunks
// K rows per chunk by config: narrow chunks for the big (throughput) tiles, whole slots for the small (latency)
// tiles so a tile is a handful of chunks.  A ring slot holds A [MTC][KC][8] then B [NTC][terms][KC][8].
// K rows per chunk: the widest chunk (so each warp's share of a chunk is a longer DMMA chain) whose ring still
// holds two slots (KW > 1) or whose slot stays <= 48 KB (KW = 1: big tiles, deeper ring).  `terms` = 2 when a
// phase has two-term panels (d + p, the op program), else 1.
__device__ __forceinline__ int cfg_kc(const TileCfg& c, int terms) {
  const int per = 128 * (c.mtc + terms * c.ntc);  // bytes per K row
  const int cap = c.kw == 1 ? 48 * 1024 : II_RING / 2;
  return per * 128 <= cap ? 128 : (per * 64 <= cap ? 64 : 32);
}
__device__ __forceinline__ uint32_t slot_elems(const TileCfg& c, int kc, int terms) {
  return (uint32_t)kc * 8u * (c.mtc + terms * c.ntc);
}

// Everything a tile's chunks need, derived once per tile (warp-uniform values).
struct TileDesc {
  int jx, job, w, nmt, ii, mt0, nt0, mvalid, nvalid, ns, nkc;
  int slots;  // slot of chunk group si in bits [2 si, 2 si + 2)
  int twos;   // bit si: two-term panel (d + p)
  int negs;   // bit si: negated panel
};

__device__ __forceinline__ TileDesc tile_desc(const InnerParams& p, const IIShared& S, const TileCfg& c, int kc,
                                              const TileRef& r, int it0) {
  TileDesc d;
  d.jx = r.jx;
  d.job = S.jjob[r.jx];
  d.w = S.jw[r.jx];
  d.nmt = (d.w + 7) >> 3;
  d.ii = it0 + r.ii;
  d.mt0 = r.mtg * c.mtc;
  d.nt0 = r.ntg * c.ntc;
  d.mvalid = min(c.mtc, d.nmt - d.mt0);
  d.nvalid = min(c.ntc, S.nact[r.jx] - d.nt0);
  d.ns = S.ins[d.ii];
  d.nkc = (d.w + kc - 1) / kc;
  const IItemS& item = S.items[d.ii];
  d.slots = d.twos = d.negs = 0;
  for (int s = 0, si = 0; s < 4; ++s)
    if (item.cell >= 0 && item.pan[s][0].vec >= 0) {
      d.slots |= s << (2 * si);
      d.twos |= (item.pan[s][1].vec >= 0) << si;
      d.negs |= (item.flags >> s & 1) << si;
      ++si;
    }
  return d;
}

// Warp 0 issues chunk (si, kcn) of tile d into a ring slot: lane a < MTC copies the Green rows of row tile
// mt0 + a, lane 8 + 2 b + t the panel term t of n-tile nt0 + b; lane 0 arms the slot's barrier with the
// chunk's byte count (complete_tx may land before the arm: the phase cannot complete while the arm's arrival
// is pending).  One round of independent bulk copies per chunk, no per-copy serial address work.
// parts: bit 0 = arm the barrier with the whole chunk's bytes and copy the Green rows (operator data, may be
// issued before the grid barrier of the phase that produces the panels), bit 1 = copy the panels.
__device__ __forceinline__ void issue_chunk_warp(const InnerParams& p, const IIShared& S, const TileCfg& c, int kc,
                                                 int terms, const TileDesc& d, int si, int kcn, double2* slotp,
                                                 uint64_t* bar, const int vmap[3], int parts = 3) {
  const int lane = threadIdx.x & 31;
  const int s = d.slots >> (2 * si) & 3, two = d.twos >> si & 1;
  const int k0 = kcn * kc, kv = min(kc, d.w - k0);
  const uint32_t bytes = (uint32_t)kv * 128u;
  if ((parts & 1) && lane == 0) mbar_expect_tx_relaxed(bar, bytes * (uint32_t)(d.mvalid + d.nvalid * (1 + two)));
  const IItemS& item = S.items[d.ii];
  if ((parts & 1) && lane < d.mvalid) {
    const long long goff = __ldg(&p.cells[S.jlay[d.jx] * p.Lc + item.cell].green_off);
    bulk_g2s(slotp + (size_t)lane * kc * 8,
             p.green + goff + ((size_t)(item.row * 4 + s) * d.nmt + d.mt0 + lane) * d.w * 8 + (size_t)k0 * 8, bytes, bar);
  } else if ((parts & 2) && lane >= 8 && lane < 8 + 2 * d.nvalid) {
    const int bq = (lane - 8) >> 1, t = (lane - 8) & 1;
    if (t <= two) {
      const RefS r = item.pan[s][t];
      const int nt = S.act[d.jx][d.nt0 + bq];
      bulk_g2s(slotp + ((size_t)c.mtc + bq * terms + t) * kc * 8,
               v2p(p, d.job, vmap[r.vec], nt) + ((size_t)r.seg * d.w + k0) * 8, bytes, bar);
    }
  }
}

// ---------------------------------------------------------------------------------------- warp product
__device__ __forceinline__ void flip_sign(double (&acc)[2][2][8]) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        acc[a][b][e] = __longlong_as_double(__double_as_longlong(acc[a][b][e]) ^ (long long)0x8000000000000000ULL);
}

// One chunk of a tile for this warp: its (WM x WN <= 2 x 2) pairs over k-steps [ks0, ks1).  wm / wn are
// warp-uniform runtime values (one code path keeps the hot loop small).
__device__ __forceinline__ void chunk_mma(const double2* A, const double2* B, int kc, int terms, int wm, int wn,
                                          int wmi, int wni, int ks0, int ks1, int kv, int two,
                                          double (&acc)[2][2][8], int mvalid, int nvalid) {
  const int lane = threadIdx.x & 31, r8 = lane >> 2, kl = lane & 3;
  const bool m1 = wm > 1 && wmi * wm + 1 < mvalid, n1 = wn > 1 && wni * wn + 1 < nvalid;
  const bool m0 = wmi * wm < mvalid, n0 = wni * wn < nvalid;
  const double2* A0 = A + (size_t)(wmi * wm) * kc * 8 + r8;
  const double2* B0 = B + (size_t)(wni * wn) * terms * kc * 8 + r8;
  const int bstride = terms * kc * 8;  // next n-tile's panel
  if (wm == 2 && wn == 2 && m1 && n1 && !two && ks1 * 4 <= kv) {
    // the common full 2 x 2 block of single-term panels over whole k-steps: no predicates, deeper unroll
#pragma unroll 4
    for (int ks = ks0; ks < ks1; ++ks) {
      const int k8 = (ks * 4 + kl) * 8;
      const double2 a0 = A0[k8], a1 = A0[kc * 8 + k8], b0 = B0[k8], b1 = B0[bstride + k8];
      dmma4(acc[0][0], a0.x, a0.y, b0.x, b0.y);
      dmma4(acc[0][1], a0.x, a0.y, b1.x, b1.y);
      dmma4(acc[1][0], a1.x, a1.y, b0.x, b0.y);
      dmma4(acc[1][1], a1.x, a1.y, b1.x, b1.y);
    }
    return;
  }
#pragma unroll 2
  for (int ks = ks0; ks < ks1; ++ks) {
    const int k = ks * 4 + kl;
    const bool kin = k < kv;
    double2 a0 = czero(), a1 = czero(), b0 = czero(), b1 = czero();
    if (kin) {
      if (m0) a0 = A0[k * 8];
      if (m1) a1 = A0[(kc + k) * 8];
      if (n0) {
        b0 = B0[k * 8];
        if (two) b0 = cadd(b0, B0[(kc + k) * 8]);  // d + p (the gather's order)
      }
      if (n1) {
        b1 = B0[bstride + k * 8];
        if (two) b1 = cadd(b1, B0[bstride + (kc + k) * 8]);
      }
    }
    dmma4(acc[0][0], a0.x, a0.y, b0.x, b0.y);
    if (wn > 1) dmma4(acc[0][1], a0.x, a0.y, b1.x, b1.y);
    if (wm > 1) {
      dmma4(acc[1][0], a1.x, a1.y, b0.x, b0.y);
      if (wn > 1) dmma4(acc[1][1], a1.x, a1.y, b1.x, b1.y);
    }
  }
}

// ---------------------------------------------------------------------------------------- program phase
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// The tile shape of a phase: minimise (tile rounds) x (cycles of one tile at its warp block's DMMA rate + a fixed
// per-tile cost).  Evaluated for every program phase when the active n-tiles change (refresh), not per phase.
__device__ __forceinline__ int phase_config(const IIShared& S, int J, int nit, int wphase, int wmax, int G,
                                            float tile_cost) {
  int cfg = II_NCFG - 1;
  const float ksteps = (float)wphase / (float)max(nit, 1) * (float)((wmax + 3) >> 2);
  float best = 3.4e38f;
  for (int ci = 0; ci < II_NCFG; ++ci) {
    const TileCfg cc = II_CFG[ci];
    const int tiles = S.tpre[ci][J] * nit;
    const int rounds = (tiles + G - 1) / G;
    const float t = (float)rounds * ((float)(cc.mtc * cc.ntc) * ksteps * 4.0f / cfg_rate(cc) + tile_cost);
    if (tiles > 0 && t < best) {
      best = t;
      cfg = ci;
    }
  }
  return cfg;
}

// Ring bookkeeping that persists across phases: consumers' full-barrier parities and the producer warp's
// empty-barrier parities, one bit per physical slot.
struct Ring {
  uint32_t fpar, epar;
  uint32_t owed;  // producer: slots holding a chunk whose release it has not waited for yet
  int pre;        // producer: chunks of the coming phase whose Green rows were issued before its grid barrier
};

// producer warp: make slot `slot` free (wait for the release of the chunk it holds, if any)
__device__ __forceinline__ void slot_claim(IIShared& S, Ring& rg, int slot) {
  if (rg.owed >> slot & 1u) {
    if ((threadIdx.x & 31) == 0) mbar_wait_suspend(&S.empty[slot], (rg.epar >> slot) & 1u);
    __syncwarp();
    rg.epar ^= 1u << slot;
  }
  rg.owed |= 1u << slot;
}

// the next phase of the same iteration (its Green rows can be prefetched across the grid barrier)
struct NextPhase {
  int it0, nit, cfg, phase_id;  // nit < 0: none
};

// One program phase over every job's active n-tiles; vmap: program vector ids {0 IN, 1 OUT, 2 AUX} ->
// scratch vector index.  Warp 0 produces (a slot is refilled once its 8 consumer warps have arrived on its
// empty barrier) and consumes like every other warp; there is no CTA-wide barrier per chunk.
__device__ __noinline__ void run_phase(const InnerParams& p, IIShared& S, double2* ring, double2* red, int J,
                                       int it0, int nit, int wphase, int pcfg, int phase_id, const int vmap[3],
                                       NextPhase nx, Ring& rg, IITick& T, IITrace& X) {
  const int tid = threadIdx.x, wp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, b = blockIdx.x;
  // ---- config: minimise (tile rounds) x (cycles of one tile at its warp block's DMMA rate + a fixed per-tile cost)
  const int cfg = pcfg;  // chosen per phase when the active sets change (phase_config)
  X.ev(20, cfg);
  const TileCfg c = II_CFG[cfg];
  const int terms = S.phtwo[phase_id] ? 2 : 1;  // two-term panels (d + p) in this phase
  const int kc = cfg_kc(c, terms), ksn = kc / 4;
  const int ntiles = S.tpre[cfg][J] * nit;
  const uint32_t se = slot_elems(c, kc, terms);
  const int nslot = min(II_NSLOT, (int)(II_RING / (se * 16u)));
  // the B panels were written by other CTAs (generic proxy) before the grid barrier; order those writes
  // before this CTA's bulk (async-proxy) reads
  if (wp == 8) asm volatile("fence.proxy.async.global;" ::: "memory");  // the producer issues the copies
  // ---- warp 8: the producer.  Walks this CTA's tiles and chunks in the consumers' order, waits for a slot's 8
  // consumer warps to release it (empty barrier), then issues the chunk's bulk copies, one lane per copy.
  if (wp == 8) {
    // chunks [0, rg.pre) were armed and their Green rows issued during the previous phase: their panels now
    int issued = 0;
    for (int t = b; t < ntiles; t += G) {
      const TileRef r = tile_decode(S, cfg, J, t);
      if (S.ins[it0 + r.ii] == 0) continue;
      const TileDesc d = tile_desc(p, S, c, kc, r, it0);
      for (int si = 0; si < d.ns; ++si)
        for (int kcn = 0; kcn < d.nkc; ++kcn) {
          const int slot = issued % nslot;
          if (issued < rg.pre) {
            issue_chunk_warp(p, S, c, kc, terms, d, si, kcn, ring + (size_t)slot * se, &S.full[slot], vmap, 2);
          } else {
            slot_claim(S, rg, slot);
            issue_chunk_warp(p, S, c, kc, terms, d, si, kcn, ring + (size_t)slot * se, &S.full[slot], vmap);
          }
          ++issued;
        }
    }
    rg.pre = 0;
    if (nx.nit > 0) {
      // every slot released (the next phase's ring layout may differ), then the next phase's first chunks: arm +
      // Green rows; their panels follow after the grid barrier
      for (int i = 0; i < II_NSLOT; ++i)
        if (rg.owed >> i & 1u) {
          if (lane == 0) mbar_wait_suspend(&S.empty[i], (rg.epar >> i) & 1u);
          __syncwarp();
          rg.epar ^= 1u << i;
        }
      rg.owed = 0;
      const TileCfg c2 = II_CFG[nx.cfg];
      const int terms2 = S.phtwo[nx.phase_id] ? 2 : 1;
      const int kc2 = cfg_kc(c2, terms2);
      const uint32_t se2 = slot_elems(c2, kc2, terms2);
      const int nslot2 = min(II_NSLOT, (int)(II_RING / (se2 * 16u)));
      const int ntiles2 = S.tpre[nx.cfg][J] * nx.nit;
      int n = 0;
      for (int t = b; t < ntiles2 && n < nslot2; t += G) {
        const TileRef r = tile_decode(S, nx.cfg, J, t);
        if (S.ins[nx.it0 + r.ii] == 0) continue;
        const TileDesc d = tile_desc(p, S, c2, kc2, r, nx.it0);
        for (int si = 0; si < d.ns && n < nslot2; ++si)
          for (int kcn = 0; kcn < d.nkc && n < nslot2; ++kcn, ++n) {
            rg.owed |= 1u << n;
            issue_chunk_warp(p, S, c2, kc2, terms2, d, si, kcn, ring + (size_t)n * se2, &S.full[n], vmap, 1);
          }
      }
      rg.pre = n;
    }
    return;
  }
  int done = 0;
  X.ev(1, cfg * 100 + nslot);
  T.tick(0);
  const int wpk = 8 / c.kw;  // warps per k part
  const int kp = wp / wpk, wq = wp - kp * wpk;
  const int wmi = wq % (c.mtc / c.wm), wni = wq / (c.mtc / c.wm);
  const int ks0 = kp * ksn / c.kw, ks1 = (kp + 1) * ksn / c.kw;  // this warp's k-steps of every chunk
  for (int t = b; t < ntiles; t += G) {
    X.ev(5, t);
    T.count(9);
    if (p.tprof && tid == 0 && b < 1024) atomicAdd(&g_ii_tiles[b], 1ULL);
    const TileDesc d = tile_desc(p, S, c, kc, tile_decode(S, cfg, J, t), it0);
    const IItemS& item = S.items[d.ii];
    const int npair = c.mtc * c.ntc;
    // combine operands of this thread's first output, fetched before the products (one output per thread covers
    // the small tiles of the latency-bound phases; larger tiles load theirs in the epilogue)
    const int o0 = tid, pr0 = o0 >> 6, pos0 = o0 & 63;
    const int ml0 = pr0 / c.ntc, nl0 = pr0 - ml0 * c.ntc, grow0 = (d.mt0 + ml0) * 8 + (pos0 >> 3);
    const bool own0 = o0 < npair * 64 && ml0 < d.mvalid && nl0 < d.nvalid && grow0 < d.w;
    const int mode = item.flags >> 8 & 3;
    double2 pre_add = czero(), pre_sub = czero(), pre_rev = czero();
    if (own0) {
      const int nt = S.act[d.jx][d.nt0 + nl0], q = pos0 & 7;
      auto opnd = [&](RefS r) { return ld_cg(v2p(p, d.job, vmap[r.vec], nt) + ((size_t)r.seg * d.w + grow0) * 8 + q); };
      if (item.add[0].vec >= 0) {
        pre_add = opnd(item.add[0]);
        if (item.add[1].vec >= 0) pre_add = cadd(pre_add, opnd(item.add[1]));
      }
      if (item.sub[0].vec >= 0) {
        pre_sub = opnd(item.sub[0]);
        if (item.sub[1].vec >= 0) pre_sub = cadd(pre_sub, opnd(item.sub[1]));
      }
      if (mode != 0) pre_rev = opnd(item.rev);
    }
    double acc[2][2][8];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[a][bb][e] = 0.0;
    for (int si = 0, q = 0; si < d.ns; ++si) {
      // a negated slot panel (exact): accumulate into -C, i.e. C - A B, by flipping the accumulators' sign bits
      // before and after the slot (integer ops: the FP64 pipe is shared with DMMA)
      const bool neg = d.negs >> si & 1;
      if (neg) flip_sign(acc);
      const int two = d.twos >> si & 1;
      for (int kcn = 0; kcn < d.nkc; ++kcn, ++q) {
        const int slot = done % nslot;
        mbar_wait_suspend(&S.full[slot], (rg.fpar >> slot) & 1u);
        rg.fpar ^= 1u << slot;
        X.ev(3, done);
        const double2* A = ring + (size_t)slot * se;
        const double2* B = A + (size_t)c.mtc * kc * 8;
        chunk_mma(A, B, kc, terms, c.wm, c.wn, wmi, wni, ks0, ks1, min(kc, d.w - kcn * kc), two, acc,
                  d.mvalid, d.nvalid);
        __syncwarp();
        // relaxed: a release arrive would first wait for every outstanding memory operation of the thread
        if (lane == 0) mbar_arrive_relaxed(&S.empty[slot]);
        ++done;
        X.ev(4, done);
      }
      if (neg) flip_sign(acc);
    }
    T.tick(1);
    // ---- partial tiles -> shared memory: red[kp][pair][row * 8 + col], pair = mtl * NTC + ntl
    if (d.ns > 0) {
      const int r8 = lane >> 2, cq = 2 * (lane & 3);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
          if (a >= c.wm || bb >= c.wn) continue;
          const int ml = wmi * c.wm + a, nl = wni * c.wn + bb;
          double2* dst = red + ((size_t)kp * npair + ml * c.ntc + nl) * 64 + r8 * 8 + cq;
          const double* q = acc[a][bb];
          dst[0] = make_double2(q[0] - q[2], q[4] + q[6]);
          dst[1] = make_double2(q[1] - q[3], q[5] + q[7]);
        }
    }
    cbar();
    // ---- combine: t = y + (add0 + add1) - (sub0 + sub1); dst = t | rev - t | t - rev
    for (int o = tid; o < npair * 64; o += II_T) {
      const int pr = o >> 6, pos = o & 63, row = pos >> 3, q = pos & 7;
      const int ml = pr / c.ntc, nl = pr - ml * c.ntc;
      const int grow = (d.mt0 + ml) * 8 + row;
      if (ml >= d.mvalid || nl >= d.nvalid || grow >= d.w) continue;
      const int nt = S.act[d.jx][d.nt0 + nl];
      double2 y = czero();
      if (d.ns > 0)
        for (int k = 0; k < c.kw; ++k) y = cadd(y, red[((size_t)k * npair + pr) * 64 + pos]);
      double2 av = pre_add, sv = pre_sub, rv = pre_rev;
      if (o != o0) {
        auto opnd = [&](RefS r) { return ld_cg(v2p(p, d.job, vmap[r.vec], nt) + ((size_t)r.seg * d.w + grow) * 8 + q); };
        av = sv = rv = czero();
        if (item.add[0].vec >= 0) {
          av = opnd(item.add[0]);
          if (item.add[1].vec >= 0) av = cadd(av, opnd(item.add[1]));
        }
        if (item.sub[0].vec >= 0) {
          sv = opnd(item.sub[0]);
          if (item.sub[1].vec >= 0) sv = cadd(sv, opnd(item.sub[1]));
        }
        if (mode != 0) rv = opnd(item.rev);
      }
      if (item.add[0].vec >= 0) y = cadd(y, av);
      if (item.sub[0].vec >= 0) y = csub(y, sv);
      if (mode == 1) y = csub(rv, y);
      else if (mode == 2) y = csub(y, rv);
      v2p(p, d.job, vmap[item.dst.vec], nt)[((size_t)item.dst.seg * d.w + grow) * 8 + q] = y;
    }
    cbar();  // red is reused by the next tile
    X.ev(6, 0);
    T.tick(2);
  }
}

// ---------------------------------------------------------------------------------------- vector phases
// Work items (job, active n-tile, element slice) of the vector phases, round-robin over the CTAs.
struct VSplit {
  int S;      // slices per (job, n-tile)
  int nitem;  // total items
};

__device__ __forceinline__ VSplit vsplit(const IIShared& S, int J, int G, int nmax_el) {
  int nv = 0;
  for (int jx = 0; jx < J; ++jx) nv += S.nact[jx];
  int sl = nv > 0 ? (G + nv - 1) / nv : 1;
  sl = max(1, min(sl, min(II_SMAX, nmax_el / 64)));
  return VSplit{sl, nv * sl};
}

__device__ __forceinline__ void vitem(const IIShared& S, int J, const VSplit& vs, int v, int& jx, int& nt, int& s) {
  s = v % vs.S;
  int k = v / vs.S;
  jx = 0;
  while (k >= S.nact[jx]) k -= S.nact[jx++];
  nt = S.act[jx][k];
}

// block reduction of per-thread values for the 8 instances: thread (e = tid >> 3, q = tid & 7); returns the
// sum for q = tid & 7 in every thread (fixed order)
__device__ __forceinline__ double2 qsum(double2 v, double* dred) {
  // lanes with the same q: xor over lane bits 3 and 4
  for (int o = 8; o < 32; o <<= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, q = threadIdx.x & 7;
  cbar();
  if (lane < 8) {
    dred[(wp * 8 + lane) * 2] = v.x;
    dred[(wp * 8 + lane) * 2 + 1] = v.y;
  }
  cbar();
  double2 s = czero();
  for (int k = 0; k < II_T / 32; ++k) s = cadd(s, make_double2(dred[(k * 8 + q) * 2], dred[(k * 8 + q) * 2 + 1]));
  return s;
}

// sum over the slices (fixed order) of partial m of instance q; vb = the work item of slice 0
__device__ __noinline__ double2 psum(const InnerParams& p, int area, int vb, int nsl, int m, int q) {
  double2 s = czero();
  int sl = 0;
  for (; sl + 4 <= nsl; sl += 4) {  // four independent loads in flight, summed in slice order
    const double2 x0 = ld_cg(partp(p, area, vb + sl) + m * 8 + q), x1 = ld_cg(partp(p, area, vb + sl + 1) + m * 8 + q);
    const double2 x2 = ld_cg(partp(p, area, vb + sl + 2) + m * 8 + q), x3 = ld_cg(partp(p, area, vb + sl + 3) + m * 8 + q);
    s = cadd(cadd(cadd(cadd(s, x0), x1), x2), x3);
  }
  for (; sl < nsl; ++sl) s = cadd(s, ld_cg(partp(p, area, vb + sl) + m * 8 + q));
  return s;
}

__device__ __forceinline__ bool inst_active(const InnerParams& p, int job, int nt, int q) {
  const int r = nt * 8 + q;
  return r < p.R && __ldcg(p.state + job * p.R + r) == 0;
}

// One (job, n-tile, element slice) item of an Arnoldi pass at step j (W = V_{j+1} holds pre(op(V_j))):
//   pass 1: h1_i = vdot(V_i, W) partials -> area 0
//   pass 2: W -= sum_i h1_i V_i (stored); h2_i = vdot(V_i, W) and ||W||^2 partials -> area 1
//   pass 3: hn^2 = ||W||^2 - ||h2||^2; W = (W - sum_i h2_i V_i) / hn (stored); owner (slice 0): column h1 + h2 | hn,
//           Givens (krylov.py:96-127), state
// Thread (e = tid >> 3, q = tid & 7) walks elements e0 + e, e0 + e + 32, ... of instance q.
__device__ __noinline__ void vec_item(const InnerParams& p, IIShared& S, int pass, int j, int job, int nt, int v, int sl, int nsl,
                         int n) {
  const int vb = v - sl;
  const int tid = threadIdx.x, q = tid & 7;
  const int e0 = (int)((long long)sl * n / nsl), e1 = (int)((long long)(sl + 1) * n / nsl);
  double2* Wp = v2p(p, job, j + 1, nt);
  const size_t hld = (size_t)p.cap + 1;
  auto V = [&](int i, int e) { return ld_cg(v2p(p, job, i, nt) + (size_t)e * 8 + q); };
  if (pass == 1 || pass == 2) {
    double2* out = partp(p, pass - 1, v);
    double nw2 = 0.0;
    for (int i0 = 0; i0 <= j; i0 += II_JREG) {
      const bool last = i0 + II_JREG > j;
      double2 h[II_JREG], acc[II_JREG];
#pragma unroll
      for (int i = 0; i < II_JREG; ++i) {
        h[i] = (pass == 2 && i0 + i <= j) ? psum(p, 0, vb, nsl, i0 + i, q) : czero();
        acc[i] = czero();
      }
      for (int e = e0 + (tid >> 3); e < e1; e += II_T / 8) {
        double2 wv = ld_cg(Wp + (size_t)e * 8 + q);
        double2 vi[II_JREG];
#pragma unroll
        for (int i = 0; i < II_JREG; ++i)
          if (i0 + i <= j) vi[i] = V(i0 + i, e);
        if (pass == 2) {
#pragma unroll
          for (int i = 0; i < II_JREG; ++i)
            if (i0 + i <= j) wv = csub(wv, cmul(h[i], vi[i]));
          Wp[(size_t)e * 8 + q] = wv;
        }
        if (pass == 1 || (last && i0 == 0))
#pragma unroll
          for (int i = 0; i < II_JREG; ++i)
            if (i0 + i <= j) acc[i] = cadd(acc[i], cconjmul(vi[i], wv));
        if (pass == 2 && last) nw2 += wv.x * wv.x + wv.y * wv.y;  // ||w'||^2 (w' is final in the last group)
      }
      if (pass == 1 || (last && i0 == 0)) {
#pragma unroll
        for (int i = 0; i < II_JREG; ++i)
          if (i0 + i <= j) {
            const double2 s2 = qsum(acc[i], S.dred);
            if (tid < 8) out[(i0 + i) * 8 + tid] = s2;
          }
      }
    }
    if (pass == 2 && j >= II_JREG) {  // more basis vectors than one register group: dots of the final w'
      for (int i = 0; i <= j; ++i) {
        double2 a = czero();
        for (int e = e0 + (tid >> 3); e < e1; e += II_T / 8) a = cadd(a, cconjmul(V(i, e), ld_cg(Wp + (size_t)e * 8 + q)));
        const double2 s2 = qsum(a, S.dred);
        if (tid < 8) out[i * 8 + tid] = s2;
      }
    }
    if (pass == 2) {
      const double2 s2 = qsum(make_double2(nw2, 0.0), S.dred);
      if (tid < 8) out[(j + 1) * 8 + tid] = s2;
    }
    return;
  }
  // pass 3.  The new basis vector is orthogonal to V to rounding after the second projection, so
  // ||w''||^2 = ||w'||^2 - ||h2||^2 (h2 = V^H w' is the reorthogonalisation correction, ~1e-16 ||w'||): the norm is
  // known before w'' is formed and the vector is stored normalised in the same pass.
  double hh = 0.0;
  const double nw2 = psum(p, 1, vb, nsl, j + 1, q).x;
  for (int i0 = 0; i0 <= j; i0 += II_JREG) {
    const bool last = i0 + II_JREG > j;
    double2 h[II_JREG];
#pragma unroll
    for (int i = 0; i < II_JREG; ++i) {
      h[i] = i0 + i <= j ? psum(p, 1, vb, nsl, i0 + i, q) : czero();
      hh += h[i].x * h[i].x + h[i].y * h[i].y;
    }
    const double hn2 = nw2 - hh;
    const double hnl = hn2 > 0.0 ? sqrt(hn2) : 0.0;
    const double ihn = (last && hnl > 0.0 && hnl < 1e300) ? 1.0 / hnl : 1.0;  // scaling by the reciprocal
    for (int e = e0 + (tid >> 3); e < e1; e += II_T / 8) {
      double2 wv = ld_cg(Wp + (size_t)e * 8 + q);
#pragma unroll
      for (int i = 0; i < II_JREG; ++i)
        if (i0 + i <= j) wv = csub(wv, cmul(h[i], V(i0 + i, e)));
      Wp[(size_t)e * 8 + q] = make_double2(wv.x * ihn, wv.y * ihn);
    }
  }
  const double hn2f = nw2 - hh;
  const double hn = hn2f > 0.0 ? sqrt(hn2f) : 0.0;
  const bool act = inst_active(p, job, nt, q);
  cbar();  // every thread has read the instance state before the owner updates it
  if (sl != 0) return;
  // owner of the (job, n-tile): stage the Hessenberg column h1 + h2 and the previous rotations of its 8
  // instances in shared memory (parallel loads), then each instance's serial rotation loop runs on thread q
  const int r_ = nt * 8;
  for (int t = tid; t < 8 * (j + 1); t += II_T) {
    const int q2 = t & 7, i = t >> 3;
    S.gv[q2][0][i] = cadd(psum(p, 0, vb, nsl, i, q2), psum(p, 1, vb, nsl, i, q2));
  }
  for (int t = tid; t < 8 * (j + 1); t += II_T) {
    const int q2 = t & 7, i = t >> 3;
    if (r_ + q2 >= p.R) continue;
    const double2* H = p.hess + (size_t)(job * p.R + r_ + q2) * p.hstride;
    const double2* g = H + hld * p.cap;
    if (i < j) {
      S.gv[q2][1][i] = ld_cg(g + (p.cap + 1) + i);      // cs[i]
      S.gv[q2][2][i] = ld_cg(g + (p.cap + 1) + p.cap + i);  // sn[i]
    } else {
      S.gv[q2][1][33] = ld_cg(g + j);  // g[j]
    }
  }
  cbar();
  if (tid < 8 && act) {
    const int r = r_ + q;
    double2* H = p.hess + (size_t)(job * p.R + r) * p.hstride;
    double2* colG = H + (size_t)j * hld;
    double2* g = H + hld * p.cap;
    double2* cs = g + (p.cap + 1);
    double2* sn = cs + p.cap;
    double2* col = S.gv[q][0];
    col[j + 1] = make_double2(hn, 0.0);
    for (int i = 0; i < j; ++i) {  // accumulated rotations (krylov.py:97-100)
      const double2 csi = S.gv[q][1][i], sni = S.gv[q][2][i];
      const double2 t = cadd(cmul(csi, col[i]), cmul(sni, col[i + 1]));
      const double2 nsc = make_double2(-sni.x, sni.y);  // -conj(sn)
      const double2 csc = make_double2(csi.x, -csi.y);  // conj(cs)
      col[i + 1] = cadd(cmul(nsc, col[i]), cmul(csc, col[i + 1]));
      col[i] = t;
    }
    const double aa = hypot(col[j].x, col[j].y);
    const double d = sqrt(aa * aa + hn * hn);
    int st = 0;  // 0 continue, 1 converged, 2 failed
    if (d == 0.0) {
      st = 2;
      atomicMax(p.err, 3);
    } else {
      const double2 c = make_double2(col[j].x / d, -col[j].y / d);
      const double2 sv = make_double2(hn / d, 0.0);
      cs[j] = c;
      sn[j] = sv;
      col[j] = cadd(cmul(c, col[j]), make_double2(sv.x * hn, 0.0));
      const double2 gj = S.gv[q][1][33];
      const double2 gj1 = cmul(make_double2(-sv.x, sv.y), gj);
      g[j + 1] = gj1;
      g[j] = cmul(c, gj);
      const double res = hypot(gj1.x, gj1.y) / __ldcg(p.beta0 + job * p.R + r);
      if (hn == 0.0) {
        st = res > p.ktol ? 2 : 1;  // happy breakdown (krylov.py:116-124)
        if (st == 2) atomicMax(p.err, 3);
      } else if (res <= p.ktol) {
        st = 1;
      } else if (j + 1 == p.max_iter) {
        st = 2;
        atomicMax(p.err, 2);  // InnerSolveError (nested.py:148-152)
      }
    }
    for (int i = 0; i <= j + 1; ++i) colG[i] = col[i];
    p.state[job * p.R + r] = st;
    if (st != 0) p.iters[job * p.R + r] = st == 1 ? j + 1 : -1;
  }
  cbar();  // S.gv is reused by the next item
}

// ---------------------------------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(II_TB, 1) inner_items_kernel(const InnerParams p, int J) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem[];
  double2* ring = reinterpret_cast<double2*>(smem);
  double2* red = reinterpret_cast<double2*>(smem + II_RING);
  IIShared& S = *reinterpret_cast<IIShared*>(smem + II_RING + II_RED);
  const int tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int nIc = p.Lc - 1;
  const int VB = p.cap + 1, VY = p.cap + 2, VT = p.cap + 3, VA = p.cap + 4;
  const int NT = (p.R + 7) >> 3;
  const size_t hld = (size_t)p.cap + 1;
  if (tid == 0) {
    for (int i = 0; i < II_NSLOT; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], II_T / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  IITick T;
  T.on = p.tprof && blockIdx.x == 0 && tid == 0;
  T.start();
  const long long t_begin = clock64();
  long long t_wait = 0;
  auto gsync = [&]() {
    const long long t0 = clock64();
    grid.sync();
    t_wait += clock64() - t0;
  };
  Ring rg{0u, 0u, 0u, 0};
  IITrace X;
  X.on = p.ii_trace > 0 && (int)blockIdx.x == p.ii_trace - 1 && tid == 0;
  X.n = 0;
  for (int jx = tid; jx < J; jx += II_TB) {
    const int job = p.stage_jobs[jx];
    S.jlay[jx] = p.jobs[job].layer;
    S.jw[jx] = p.layers[S.jlay[jx]].w;
    S.jjob[jx] = job;
  }
  S.gv = reinterpret_cast<double2(*)[3][34]>(red);
  S.yv = reinterpret_cast<double2(*)[34]>(red + 8 * 3 * 34);
  for (int i = tid; i < p.nitems; i += II_TB) {
    S.items[i] = pack_item(p.items[i]);
    S.ins[i] = (unsigned char)item_ns_g(p.items[i]);
  }
  __syncthreads();
  for (int ph = tid; ph < p.op_nph + p.pre_nph; ph += II_TB) {
    const int* phd = ph < p.op_nph ? p.op_ph + ph : p.pre_ph + (ph - p.op_nph);
    int wsum = 0, two = 0;
    for (int i = phd[0]; i < phd[1]; ++i) {
      wsum += S.ins[i] > 0 ? S.ins[i] : 1;
      for (int s_ = 0; s_ < 4; ++s_) two |= S.items[i].cell >= 0 && S.items[i].pan[s_][1].vec >= 0;
    }
    S.phw[ph] = wsum;
    S.phtwo[ph] = (unsigned char)two;
  }
  // active n-tiles: all == every existing instance (before the states exist)
  auto refresh = [&](bool all) {
    __syncthreads();
    for (int t = tid; t < J * NT; t += II_TB) {
      const int jx = t / NT, nt = t - jx * NT, job = S.jjob[jx];
      unsigned m = 0;
      for (int q = 0; q < 8; ++q) {
        const int r = nt * 8 + q;
        if (r < p.R && (all || __ldcg(p.state + job * p.R + r) == 0)) m |= 1u << q;
      }
      S.amask[jx][nt] = (unsigned char)m;
    }
    __syncthreads();
    if (tid == 0) {
      int any = 0;
      for (int jx = 0; jx < J; ++jx) {
        int na = 0;
        for (int nt = 0; nt < NT; ++nt)
          if (S.amask[jx][nt]) S.act[jx][na++] = (unsigned char)nt;
        S.nact[jx] = na;
        any |= na;
      }
      S.any_active = any;
      for (int ci = 0; ci < II_NCFG; ++ci) {
        int acc = 0;
        for (int jx = 0; jx < J; ++jx) {
          S.tpre[ci][jx] = acc;
          const Geo g = job_geo(S, II_CFG[ci], jx);
          acc += g.nmtg * g.nntg;
        }
        S.tpre[ci][J] = acc;
      }
    }
    __syncthreads();
    for (int ph = tid; ph < p.op_nph + p.pre_nph; ph += II_TB) {
      const int* phd = ph < p.op_nph ? p.op_ph + ph : p.pre_ph + (ph - p.op_nph);
      S.phcfg[ph] = (unsigned char)phase_config(S, J, phd[1] - phd[0], S.phw[ph], p.wmax, G,
                                                 p.ii_tilecost > 0 ? (float)p.ii_tilecost : 3000.0f);
    }
    __syncthreads();
  };
  // one program; `then_pre`: the preconditioner program follows in the same iteration (its first phase's Green
  // rows are prefetched across the op program's last grid barrier)
  auto program = [&](const int* ph_d, int nph, int phw0, const int vm[3], bool then_pre) {
    for (int phz = 0; phz < nph; ++phz) {
      const int i0 = ph_d[phz], i1 = ph_d[phz + 1];
      NextPhase nx{0, -1, 0, 0};
      if (phz + 1 < nph) {
        nx = NextPhase{ph_d[phz + 1], ph_d[phz + 2] - ph_d[phz + 1], S.phcfg[phw0 + phz + 1], phw0 + phz + 1};
      } else if (then_pre) {
        nx = NextPhase{p.pre_ph[0], p.pre_ph[1] - p.pre_ph[0], S.phcfg[p.op_nph], p.op_nph};
      }
      run_phase(p, S, ring, red, J, i0, i1 - i0, S.phw[phw0 + phz], S.phcfg[phw0 + phz], phw0 + phz, vm, nx, rg, T, X);
      T.count(8);
      X.ev(7, phz);
      gsync();
      X.ev(8, phz);
      T.tick(3);
    }
  };
  // ---- rhs_pol from the Newton tables (sie.py:230-242, negated) into VB, padding instances zero
  {
    for (int jx = 0; jx < J; ++jx) {
      const int job = S.jjob[jx], w = S.jw[jx], n = 4 * nIc * w;
      const long long tot = (long long)NT * n * 8;
      double2* vb = v2p(p, job, VB, 0);
      for (long long t = (long long)b * II_T + tid; tid < II_T && t < tot; t += (long long)G * II_T) {
        const int q = (int)(t & 7);
        const long long rest = t >> 3;
        const int nt = (int)(rest / n), e = (int)(rest - (long long)nt * n);
        const int r = nt * 8 + q;
        double2 v = czero();
        if (r < p.R) {
          const int seg = e / w, jj = e - seg * w;
          const int half = seg / (2 * nIc);
          const int I = (seg % (2 * nIc)) / 2, s_ = seg & 1;
          const int cc = half == 0 ? I : I + 1;
          const int idx = half == 0 ? 2 + s_ : s_;
          const double2 tv = __ldcg(p.tables + ((((size_t)job * p.Lc + cc) * 4 + idx) * p.R + r) * p.wmax + jj);
          v = make_double2(-tv.x, -tv.y);
        }
        vb[((size_t)nt * p.nmax + e) * 8 + q] = v;
      }
    }
  }
  refresh(true);
  T.tick(4);
  gsync();
  T.tick(5);
  // ---- b = pre(rhs) (krylov.py:61)
  {
    const int vm[3] = {VB, VY, VA};
    program(p.pre_ph, p.pre_nph, p.op_nph, vm, false);
  }
  // ---- beta0 = ||b||, V_0 = b / beta0, g[0] = beta0 (krylov.py:63-86)
  {
    const VSplit vs = vsplit(S, J, G, 4 * nIc * p.wmax);
    for (int v = b; tid < II_T && v < vs.nitem; v += G) {
      int jx, nt, sl;
      vitem(S, J, vs, v, jx, nt, sl);
      const int job = S.jjob[jx], n = 4 * nIc * S.jw[jx];
      const int e0 = (int)((long long)sl * n / vs.S), e1 = (int)((long long)(sl + 1) * n / vs.S);
      const double2* Y = v2p(p, job, VY, nt);
      double ss = 0.0;
      for (int e = e0 + (tid >> 3); e < e1; e += II_T / 8) {
        const double2 y = ld_cg(Y + (size_t)e * 8 + (tid & 7));
        ss += y.x * y.x + y.y * y.y;
      }
      const double2 s2 = qsum(make_double2(ss, 0.0), S.dred);
      if (tid < 8) partp(p, 0, v)[tid] = s2;
    }
    T.tick(4);
    gsync();
    T.tick(5);
    for (int v = b; tid < II_T && v < vs.nitem; v += G) {
      int jx, nt, sl;
      vitem(S, J, vs, v, jx, nt, sl);
      const int job = S.jjob[jx], n = 4 * nIc * S.jw[jx];
      const int e0 = (int)((long long)sl * n / vs.S), e1 = (int)((long long)(sl + 1) * n / vs.S);
      const int q = tid & 7;
      const double b0 = sqrt(psum(p, 0, v - sl, vs.S, 0, q).x);
      const double ib0 = b0 != 0.0 ? 1.0 / b0 : 0.0;
      const double2* Y = v2p(p, job, VY, nt);
      double2* V0 = v2p(p, job, 0, nt);
      for (int e = e0 + (tid >> 3); e < e1; e += II_T / 8) {
        const double2 y = ld_cg(Y + (size_t)e * 8 + q);
        V0[(size_t)e * 8 + q] = make_double2(y.x * ib0, y.y * ib0);
      }
      const int r = nt * 8 + q;
      if (sl == 0 && tid < 8 && r < p.R) {
        double2* g = p.hess + (size_t)(job * p.R + r) * p.hstride + hld * p.cap;
        g[0] = make_double2(b0, 0.0);
        p.beta0[job * p.R + r] = b0;
        p.state[job * p.R + r] = b0 == 0.0 ? 1 : 0;
        p.iters[job * p.R + r] = b0 == 0.0 ? 0 : -1;
      }
    }
    T.tick(4);
    gsync();
    T.tick(5);
  }
  // ---- Arnoldi iterations (krylov.py:88-127)
  for (int j = 0; j < p.max_iter; ++j) {
    refresh(false);
    if (!S.any_active) break;
    if (j + 1 > p.cap) {  // basis capacity exhausted: the host retries with a larger capacity
      for (int t = b * II_T + tid; tid < II_T && t < J * p.R; t += G * II_T) {
        const int jx = t / p.R, r = t - jx * p.R, job = S.jjob[jx];
        if (__ldcg(p.state + job * p.R + r) == 0) {
          p.state[job * p.R + r] = 2;
          p.iters[job * p.R + r] = -1;
          atomicMax(p.err, 5);
        }
      }
      T.tick(4);
      gsync();
      T.tick(5);
      break;
    }
    {
      const int vm1[3] = {j, VT, VA};
      program(p.op_ph, p.op_nph, 0, vm1, true);  // VT = op(V_j)
      const int vm2[3] = {VT, j + 1, VA};
      program(p.pre_ph, p.pre_nph, p.op_nph, vm2, false);  // V_{j+1} = w = pre(op(V_j))
    }
    const VSplit vs = vsplit(S, J, G, 4 * nIc * p.wmax);
    // pass 1: h1_i = vdot(V_i, w), i <= j -> area 0
    for (int v = b; tid < II_T && v < vs.nitem; v += G) {
      int jx, nt, sl;
      vitem(S, J, vs, v, jx, nt, sl);
      vec_item(p, S, 1, j, S.jjob[jx], nt, v, sl, vs.S, 4 * nIc * S.jw[jx]);
    }
    T.tick(4);
    gsync();
    T.tick(5);
    // pass 2: w' = w - V h1 (stored), h2_i = vdot(V_i, w') and ||w'||^2 -> area 1
    for (int v = b; tid < II_T && v < vs.nitem; v += G) {
      int jx, nt, sl;
      vitem(S, J, vs, v, jx, nt, sl);
      vec_item(p, S, 2, j, S.jjob[jx], nt, v, sl, vs.S, 4 * nIc * S.jw[jx]);
    }
    T.tick(4);
    gsync();
    T.tick(5);
    // pass 3: V_{j+1} = (w' - V h2) / hn with hn^2 = ||w'||^2 - ||h2||^2; the Hessenberg column h1 + h2, hn and the
    // Givens step of every active instance on the owner (slice 0) of its (job, n-tile)
    for (int v = b; tid < II_T && v < vs.nitem; v += G) {
      int jx, nt, sl;
      vitem(S, J, vs, v, jx, nt, sl);
      vec_item(p, S, 3, j, S.jjob[jx], nt, v, sl, vs.S, 4 * nIc * S.jw[jx]);
    }
    T.tick(4);
    gsync();
    T.tick(5);
  }
  // ---- x = V_k y (back substitution), traces = down + up (nested.py:153), accounting (nested.py:54-73)
  refresh(true);
  {
    const VSplit vs = vsplit(S, J, G, 2 * nIc * p.wmax);
    for (int v = b; tid < II_T && v < vs.nitem; v += G) {
      int jx, nt, sl;
      vitem(S, J, vs, v, jx, nt, sl);
      const int job = S.jjob[jx], w = S.jw[jx], half = 2 * nIc * w;
      const int q = tid & 7, r = nt * 8 + q;
      cbar();
      // the triangle H[0..k)[0..k) and g[0..k) of the 8 instances staged in shared memory (k <= 12: packed
      // column-major after g in S.gv[q]), then the back substitution runs on thread q without L2 round trips
      if (tid < 8) S.yv[tid][33] = make_double2((double)(nt * 8 + tid < p.R ? max(0, __ldcg(p.iters + job * p.R + nt * 8 + tid)) : 0), 0.0);
      cbar();
      for (int t = tid; t < 8 * 102; t += II_T) {
        const int q2 = t / 102, e = t - q2 * 102;
        const int k2 = (int)S.yv[q2][33].x;
        if (k2 > 12 || nt * 8 + q2 >= p.R) continue;
        const double2* H = p.hess + (size_t)(job * p.R + nt * 8 + q2) * p.hstride;
        double2* dst = &S.gv[q2][0][0] + e;
        if (e < k2) {
          *dst = ld_cg(H + hld * p.cap + e);  // g[e]
        } else if (e - k2 < k2 * (k2 + 1) / 2) {
          const int f = e - k2;
          int m = 0;
          while ((m + 1) * (m + 2) / 2 <= f) ++m;
          *dst = ld_cg(H + (size_t)m * hld + (f - m * (m + 1) / 2));  // H[i][m], i = f - m(m+1)/2
        }
      }
      cbar();
      if (tid < 8) {
        const int k = (int)S.yv[q][33].x;
        const bool sm = k <= 12;
        const double2* H = p.hess + (size_t)(job * p.R + (r < p.R ? r : 0)) * p.hstride;
        const double2* g = H + hld * p.cap;
        const double2* gs = &S.gv[q][0][0];
        const double2* hs = gs + k;
        for (int i = k - 1; i >= 0; --i) {
          double2 sacc = czero();
          for (int m = i + 1; m < k; ++m) cfma(sacc, sm ? hs[m * (m + 1) / 2 + i] : H[(size_t)m * hld + i], S.yv[q][m]);
          const double2 num = csub(sm ? gs[i] : g[i], sacc);
          const double2 den = sm ? hs[i * (i + 1) / 2 + i] : H[(size_t)i * hld + i];
          const double dd = den.x * den.x + den.y * den.y;
          S.yv[q][i] = make_double2((num.x * den.x + num.y * den.y) / dd, (num.y * den.x - num.x * den.y) / dd);
        }
        if (sl == 0 && r < p.R) {
          atomicAdd(&p.hist[min(k, PT_HIST - 1)], 1);
          atomicAdd(&p.counters[0], (unsigned long long)k);
          const unsigned long long t =
              ((unsigned long long)(k + 1) * p.pre_blocks + (unsigned long long)k * p.op_blocks) * w * w;
          atomicAdd(&p.counters[1], t);
          atomicAdd(&p.counters[2], 1ULL);
        }
      }
      cbar();
      const int k = (int)S.yv[q][33].x;
      const int e0 = (int)((long long)sl * half / vs.S), e1 = (int)((long long)(sl + 1) * half / vs.S);
      double2* out = p.tr + (size_t)(job * p.R + (r < p.R ? r : 0)) * nIc * 2 * p.wmax;
      for (int e = e0 + (tid >> 3); e < e1; e += II_T / 8) {
        double2 xd = czero(), xu = czero();
        for (int i = 0; i < k; ++i) {
          const double2* Vi = v2p(p, job, i, nt);
          cfma(xd, ld_cg(Vi + (size_t)e * 8 + q), S.yv[q][i]);
          cfma(xu, ld_cg(Vi + (size_t)(half + e) * 8 + q), S.yv[q][i]);
        }
        const int seg = e / w, jj = e - seg * w;
        if (r < p.R) out[(size_t)seg * p.wmax + jj] = cadd(xd, xu);
      }
    }
  }
  T.tick(7);
  X.ev(15, 0);
  if (X.on && X.n < II_NEV) g_ii_ev[X.n] = 0;
  if (p.tprof && tid == 0 && b < 1024) g_ii_w[b] += (unsigned long long)(clock64() - t_begin - t_wait);
}

// ---------------------------------------------------------------------------------------- launcher
long long inner_items_part_items(int num_sms, int jmax, int rmax) {
  return (long long)num_sms + (long long)jmax * ((rmax + 7) / 8);
}

static_assert(II_RING + II_RED + sizeof(IIShared) <= 232448, "inner_items_kernel exceeds 227 KB of shared memory");

cudaError_t inner_items_launch(const InnerParams& p0, int J, cudaStream_t st) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  static const bool v1 = std::getenv("PT_ITEMS_V1") != nullptr;  // the per-8-RHS-unit kernel instead
  // a single-job stage with one n-tile of RHS (a 1-RHS sweep stage) runs here with the scan form of the sweeps
  // (cfg5 1 RHS: 998 ms per solve against 1180 ms on the per-8-RHS-unit kernel, 8 RHS 1071 against 1305 ms);
  // without the scan program the per-8-RHS-unit kernel's per-phase latency is lower (1343 ms here), and that
  // kernel with the scan program is slower still (2202 ms: its unit-major split serialises the levels' items):
  // PT_ITEMS_ALL=1 selects this kernel for every stage regardless
  static const bool all = std::getenv("PT_ITEMS_ALL") != nullptr;
  const bool scan = p0.pre_nph_px > 0 && p0.items_px && p0.nitems_px <= II_MAXIT;
  if (v1 || (!all && !scan && J < 2 && p0.R <= 8) || p0.dense || !p0.part || J < 1 || J > II_MAXJ || p0.R > II_MAXNT * 8 || p0.cap > 32 || p0.Lc < 2 ||
      p0.nitems > II_MAXIT || p0.op_nph + p0.pre_nph > II_MAXPH ||
      p0.part_items < inner_items_part_items(nsm, J, p0.R))
    return cudaErrorNotSupported;
  InnerParams p = p0;
  // single-job stages (the sequential outer sweeps): the scan form of the GS sweeps, 2 ceil(log2 nI) + 1
  // phases per preconditioner application instead of 2 nI - 1, up to 128 RHS (PT_SCAN_MAXR): beyond, the phases of
  // the sequential program are throughput-sized themselves and the scan's 1.7x flops cost more than its barriers
  // save (cfg4, 256 RHS in one batch: 3449 ms sequential against 3548 ms; 128 RHS: 2022 against 1994 ms)
  static const int scan_maxr = std::getenv("PT_SCAN_MAXR") ? atoi(std::getenv("PT_SCAN_MAXR")) : 128;
  if (J == 1 && p.pre_nph_px > 0 && p.items_px && p.R <= scan_maxr && p.nitems_px <= II_MAXIT) {
    p.items = p.items_px;
    p.pre_ph = p.pre_ph_px;
    p.pre_nph = p.pre_nph_px;
    p.nitems = p.nitems_px;
  }
  const int NT = (p.R + 7) / 8;
  p.s2_vec = (long long)NT * p.nmax * 8;
  p.s2_job = (long long)(p.cap + 5) * p.s2_vec;
  const size_t sm = (size_t)II_RING + II_RED + sizeof(IIShared);
  set_smem_attr((const void*)inner_items_kernel, sm);
  static int per_sm = -1;
  if (per_sm < 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inner_items_kernel, II_TB, sm);
    cudaGetLastError();
  }
  if (per_sm < 1) return cudaErrorNotSupported;
  int j_ = J;
  void* args[] = {(void*)&p, (void*)&j_};
  const int grid = p.coop_sms > 0 ? std::min(nsm, p.coop_sms) : nsm;
  return cudaLaunchCooperativeKernel((const void*)inner_items_kernel, dim3(grid), dim3(II_TB), args, sm, st);
}

void inner_items_trace_dump(const char* tag) {
  static int dumped = 0;
  if (dumped || std::strcmp(tag, "sdown") != 0) return;
  static int seen = 0;
  if (++seen < 40) return;  // a warm sweep stage
  dumped = 1;
  static unsigned long long ev[II_NEV];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(ev, g_ii_ev, sizeof(ev));
  unsigned t0 = (unsigned)(ev[0] & 0xffffffffu);
  fprintf(stderr, "items trace [%s]:", tag);
  for (int i = 0; i < II_NEV && ev[i]; ++i) {
    const unsigned t = (unsigned)(ev[i] & 0xffffffffu);
    fprintf(stderr, " %d/%d@%u", (int)(ev[i] >> 56), (int)((ev[i] >> 32) & 0xffffff), t - t0);
  }
  fprintf(stderr, "\n");
}

void inner_items_tprof_dump(const char* tag) {
  inner_items_trace_dump(tag);
  unsigned long long t[16];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(t, g_ii_t, sizeof(t));
  if (t[8] == 0 && t[9] == 0) return;
  fprintf(stderr,
          "items tprof [%s] (cycles, CTA 0): setup %llu chunks %llu epilogue %llu phase-bar %llu | vector %llu "
          "vector-bar %llu | final %llu | phases %llu tiles %llu | issue-block %llu fullwait %llu mma %llu issue %llu "
          "chunkn %llu\n",
          tag, t[0], t[1], t[2], t[3], t[4], t[5], t[7], t[8], t[9], t[10], t[11], t[12], t[13], t[14]);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_ii_t, z, sizeof(z));
  static unsigned long long w[1024];
  cudaMemcpyFromSymbol(w, g_ii_w, sizeof(w));
  unsigned long long mx = 0, sum = 0;
  int n = 0, amx = 0;
  for (int i = 0; i < 1024; ++i)
    if (w[i]) {
      if (w[i] > mx) {
        mx = w[i];
        amx = i;
      }
      sum += w[i];
      ++n;
    }
  fprintf(stderr, "items ctawork [%s] (cycles outside grid barriers): cta0 %llu mean %llu max %llu (cta %d) over %d ctas\n",
          tag, w[0], n ? sum / n : 0ULL, mx, amx, n);
  static unsigned long long tl[1024];
  cudaMemcpyFromSymbol(tl, g_ii_tiles, sizeof(tl));
  if (std::getenv("PT_INNER_TPROF_CTAS")) {
    fprintf(stderr, "items ctas [%s] work(kcycles)/tiles:", tag);
    for (int i = 0; i < n; ++i) fprintf(stderr, " %d:%llu/%llu", i, w[i] / 1000, tl[i]);
    fprintf(stderr, "\n");
  }
  memset(tl, 0, sizeof(tl));
  cudaMemcpyToSymbol(g_ii_tiles, tl, sizeof(tl));
  memset(w, 0, sizeof(w));
  cudaMemcpyToSymbol(g_ii_w, w, sizeof(w));
}
