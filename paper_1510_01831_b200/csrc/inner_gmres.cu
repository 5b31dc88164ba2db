// Inner polarized-traces GMRES (replaces _InnerPT.solve_traces, nested.py:134-153).
//
// One thread-block CLUSTER (INNER_CS CTAs) per (layer-solve job, group of up to 8
// right-hand-side instances).  The instances of a group advance in lockstep and
// are frozen individually when they converge, so every instance runs exactly the
// Krylov process of krylov.gmres (krylov.py:53-135): same operator (inner
// apply_M_polarized on the dense Green blocks, sie.py:203-228 /
// nested.py:113-122), same left GS preconditioner (sie.py:272-326), MGS Arnoldi
// with vdot, complex Givens, stop when |g_{j+1}|/beta0 <= inner_ktol, x = V_k y.
// The data-dependent iteration count never leaves the device.
//
// Operator and preconditioner run from host-built "item programs": one item is
// one sampled panel  sum_slot G[cell][row][slot] @ panel_slot + add - (sub0+sub1),
// i.e. exactly the arithmetic of the reference's TraceSystem methods; the items
// of a phase are independent and phases are separated by cluster barriers.
// A work unit is (item, group of two 8-row tiles of the output panel): its Green
// tiles (stored tile-major, [row tile][k][8 rows], so one tile is one contiguous
// bulk copy) arrive by cp.async.bulk on an mbarrier while the CTA gathers the
// slot panels, and the product runs on the FP64 tensor cores (mma.sync m8n8k4,
// SASS DMMA) with the group's 8 instances as the N dimension.  Arnoldi, Givens
// and x = V y of an instance run on one CTA of the cluster, so reductions are
// deterministic and need no cross-CTA traffic.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "pt_launch.cuh"
#include "stage_dev.cuh"

namespace cg = cooperative_groups;

#define IN_MG 2   // max 8-row tiles per group (2 for w <= 80, else 1)
#define IN_THREADS 256
#define IN_TRMAX 16  // max Green-tile ring slots of the item-program path

__device__ __forceinline__ double2* vecp(const InnerParams& p, int job, int r, int v) {
  return p.scratch + (size_t)(job * p.R + r) * p.inst_stride + (size_t)v * p.nmax;
}

__device__ __forceinline__ void csync() { cg::this_cluster().sync(); }

// optional clock64 segment totals (PT_INNER_TPROF): 0 tile issue+add/sub prefetch, 1 panel gather,
// 2 tile wait, 3 dmma, 4 combine, 5 cluster barriers, 6 arnoldi+givens, 7 rest
__device__ long long g_in_t[16];  // 8 setup, 9 final x = V y, 10 programs run, 11 kernel total
struct Ticker {
  bool on;
  long long t0;
  __device__ void start() {
    if (on) t0 = clock64();
  }
  __device__ void tick(int i) {
    if (on) {
      const long long t = clock64();
      atomicAdd((unsigned long long*)&g_in_t[i], (unsigned long long)(t - t0));
      t0 = t;
    }
  }
};

struct InSmem {
  double2* tiles;   // [p.tring][w][8] ring of single Green tiles
  double2* pan;     // [4 slots][w][8]
  double2* pan2;    // [2][w][8] second terms of two-term panels
  double2* red;     // [8 warps][IN_MG*8][8]
  uint64_t* tbar;   // [IN_TRMAX] one mbarrier per tile ring slot
  int* act;         // active local instances
  IItem* items;     // the op + pre programs (staged once)
  long long* goff;  // [Lc] Green-pool offsets of this layer's cells (staged once)
  int* oph;         // op program phase offsets (staged once)
  int* pph;         // pre program phase offsets (staged once)
  uint64_t* dbar;   // [2 * DA_NS] dense-apply ring barriers: full[DA_NS], empty[DA_NS]
  size_t region;    // bytes from tiles to the end of red (the dense-apply ring lives there)
};

// Issue (thread 0) the first min(tring, tiles) Green tiles of a future item_unit call with the same tile order
// and ring sequence numbers (from *tseq) that item_unit uses; returns how many were issued.  The tiles are
// operator data, independent of the phase results, so they can be in flight across the grid barrier.
__device__ int item_prefetch(const InnerParams& p, int w, const IItem& item, int g0, int g1, const InSmem& S,
                             const uint32_t* tseq, long long goff) {
  const int nmt = (w + 7) >> 3, MG = p.mg, TR = p.tring;
  int slotp = 0, ns = 0;
  if (item.cell >= 0)
    for (int s_ = 0; s_ < 4; ++s_)
      if (item.pan[s_][0].vec >= 0) slotp |= s_ << (2 * ns++);
  if (ns == 0) return 0;
  int ntl = 0;
  for (int g = g0; g < g1; ++g) ntl += ns * min(MG, nmt - g * MG);
  const int n = min(TR, ntl);
  const uint32_t tbytes = (uint32_t)w * 8u * 16u;
  for (int j = 0; j < n; ++j) {
    const int per = ns * MG;
    const int g = g0 + j / per;
    const int nt = min(MG, nmt - g * MG), rem = j - (j / per) * per;
    const int si = rem / nt, t = rem - si * nt;
    const uint32_t sq = *tseq + (uint32_t)j;
    const int slot = (int)(sq % (uint32_t)TR);
    mbar_expect_tx(&S.tbar[slot], tbytes);
    bulk_g2s(S.tiles + (size_t)slot * w * 8,
             p.green + goff + ((size_t)(item.row * 4 + (slotp >> (2 * si) & 3)) * nmt + g * MG + t) * w * 8, tbytes,
             &S.tbar[slot]);
  }
  return n;
}

// One unit of a program phase: item `item` over its tile groups [g0, g1), for the nact active instances
// act[0..nact) (local ids from r0) of job `job` (layer width w, Green pool offset goff of the item's cell).
// Gathers the item's panels, streams its Green tiles through the ring, runs the DMMA products and writes the
// combined outputs.  Used by the cluster kernel (run_program) and the cooperative item kernel.
__device__ void item_unit(const InnerParams& p, int job, int w, int r0, const int* act, int nact, const IItem& item,
                          int g0, int g1, const int vmap[3], const InSmem& S, uint32_t* tseq, Ticker& T, long long goff,
                          int pre = 0) {
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int nmt = (w + 7) >> 3;
  const int MG = p.mg;
  const int kps = (w + 3) >> 2;  // k-steps per slot
  const uint32_t tbytes = (uint32_t)w * 8u * 16u;
  auto VM = [&](int i) { return i == 0 ? vmap[0] : (i == 1 ? vmap[1] : vmap[2]); };
  int slotp = 0, ns = 0;  // packed slot list: slot of si in bits [2si, 2si+2)
  if (item.cell >= 0)
    for (int s = 0; s < 4; ++s)
      if (item.pan[s][0].vec >= 0) slotp |= s << (2 * ns++);
  auto slot_of = [&](int si) { return slotp >> (2 * si) & 3; };
  // The unit's Green tiles stream through a ring of p.tring single-tile slots (one 8-row tile of one slot
  // block per copy, so the ring fits any w <= 128): local tile j = (group g0 + j / (ns MG), then slot-major
  // (si, t) within the group).  tseq counts this CTA's tiles across units and programs (slot tseq % TR,
  // mbarrier parity (tseq / TR) & 1).  Issued by lane 0 of warp 0; consumers release a slot at the
  // __syncthreads that ends its tile.
  const int TR = p.tring;
  auto tile_of = [&](int j, int& g, int& si, int& t) {
    const int per = ns * MG;
    g = g0 + j / per;
    const int mt0 = g * MG, nt = min(MG, nmt - mt0), rem = j - (j / per) * per;
    si = rem / nt;
    t = rem - si * nt;
  };
  int ntl = 0;
  for (int g = g0; g < g1; ++g) ntl += ns * min(MG, nmt - g * MG);
  const uint32_t tbase = *tseq;
  int ji = 0;  // tiles issued so far (thread 0's count; ring holds tiles [jt, ji))
  auto issue_tile = [&](int j) {  // lane 0 of warp 0 only
    int g, si, t;
    tile_of(j, g, si, t);
    const uint32_t sq = tbase + (uint32_t)j;
    const int slot = (int)(sq % (uint32_t)TR);
    mbar_expect_tx(&S.tbar[slot], tbytes);
    bulk_g2s(S.tiles + (size_t)slot * w * 8,
             p.green + goff + ((size_t)(item.row * 4 + slot_of(si)) * nmt + g * MG + t) * w * 8, tbytes,
             &S.tbar[slot]);
  };
  int negm = 0;  // bit si: slot panel si enters negated (exact)
  for (int si = 0; si < ns; ++si) negm |= (item.flags >> slot_of(si) & 1) << si;
  int twom = 0;  // bit si: two-term slot panel (d + p); its second term is staged in pan2
  for (int si = 0; si < ns; ++si) twom |= (item.pan[slot_of(si)][1].vec >= 0) << si;
  if (ns > 0) {
    if (tid == 0)
      for (int j = pre; j < min(TR, ntl); ++j) issue_tile(j);  // [0, pre) came with a prefetch
    ji = min(TR, ntl);
    T.tick(13);  // tile issue
    // slot panels as B fragments pan[si][k][qq] (16-byte cp.async, inactive instances zero-fill).
    // IN_THREADS % 8 == 0, so a thread's instance qq is fixed and its scratch base is computed once.
    const int qq = tid & 7;
    const bool okq = qq < nact;
    const double2* ibase = p.scratch + (size_t)(job * p.R + (okq ? r0 + act[qq] : r0)) * p.inst_stride;
    for (int si = 0, n2 = 0; si < ns; ++si) {
      const Ref pr = item.pan[slot_of(si)][0], pr2 = item.pan[slot_of(si)][1];
      const double2* src = ibase + (size_t)VM(pr.vec) * p.nmax + pr.seg * w;
      double2* dst = S.pan + (size_t)si * w * 8 + qq;
      for (int k = tid >> 3; k < w; k += IN_THREADS / 8) cp_async16(dst + k * 8, src + k, okq);
      if (pr2.vec >= 0) {
        const double2* src2 = ibase + (size_t)VM(pr2.vec) * p.nmax + pr2.seg * w;
        double2* dst2 = S.pan2 + (size_t)n2++ * w * 8 + qq;
        for (int k = tid >> 3; k < w; k += IN_THREADS / 8) cp_async16(dst2 + k * 8, src2 + k, okq);
      }
    }
  }
  T.tick(0);
  int jt = 0;  // next local tile to consume
  for (int g = g0; g < g1; ++g) {
    const int mt0 = g * MG, nt = min(MG, nmt - mt0);
    const int row0 = mt0 * 8, rows = min(w, row0 + nt * 8) - row0;
    // this thread's output (row, instance) and its combine operands
    const int oq = tid & 7, orow = tid >> 3;
    const bool own = orow < rows && oq < nact;
    const int rr = own ? r0 + act[oq] : r0;
    const int gi = row0 + orow;
    double2 addv = czero(), subv = czero(), revv = czero();
    if (own) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (item.add[t].vec >= 0) addv = cadd(addv, ld_cg(vecp(p, job, rr, VM(item.add[t].vec)) + item.add[t].seg * w + gi));
        if (item.sub[t].vec >= 0) subv = cadd(subv, ld_cg(vecp(p, job, rr, VM(item.sub[t].vec)) + item.sub[t].seg * w + gi));
      }
      if (item.rev.vec >= 0) revv = ld_cg(vecp(p, job, rr, VM(item.rev.vec)) + item.rev.seg * w + gi);
    }
    double2 y = czero();
    if (ns > 0) {
      if (g == g0) {
        cp_async_wait_all();
        __syncthreads();
      }
      T.tick(1);
      // The group's P = ns x nt tiles are all in the ring at once (TR >= 4 MG); warp wp takes tile
      // q = wp % P (slot si = q / nt, row tile t = q % nt) and k-part wp / P of KP = 8 / P parts, so every
      // warp runs one long independent DMMA chain and the CTA synchronises once per group:
      // Cr += Ar Br + (-Ai) Bi, Ci += Ar Bi + Ai Br
      const int P = ns * nt, KP = (IN_THREADS / 32) / P;
      const int ar = lane >> 2, ak = lane & 3;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
      if (wp < P * KP) {
        const int q = wp % P, kp = wp / P;
        const int si = q / nt;
        const uint32_t sq = tbase + (uint32_t)(jt + q);
        const int slot = (int)(sq % (uint32_t)TR);
        const double sg = (negm >> si & 1) ? -1.0 : 1.0;
        const bool two = twom >> si & 1;
        const int i2 = __popc(twom & ((1 << si) - 1));
        mbar_wait(&S.tbar[slot], (sq / (uint32_t)TR) & 1);
        const double2* tl = S.tiles + (size_t)slot * w * 8;
        const int kb = kp * kps / KP, ke = (kp + 1) * kps / KP;
#pragma unroll 4
        for (int ks = kb; ks < ke; ++ks) {
          const int k = ks * 4 + ak;
          const bool kin = k < w;
          double2 bv = kin ? S.pan[((size_t)si * w + k) * 8 + ar] : czero();
          if (two) bv = cadd(bv, kin ? S.pan2[((size_t)i2 * w + k) * 8 + ar] : czero());  // d + p
          bv.x *= sg;
          bv.y *= sg;
          const double2 av = kin ? tl[(size_t)k * 8 + ar] : czero();
          dmma_f64(c0, c1, av.x, bv.x);
          dmma_f64(c2, c3, av.x, bv.y);
          dmma_f64(c0, c1, -av.y, bv.y);
          dmma_f64(c2, c3, av.y, bv.x);
        }
      }
      T.tick(2);
      S.red[((wp * IN_MG) * 8 + ar) * 8 + 2 * ak] = make_double2(c0, c2);
      S.red[((wp * IN_MG) * 8 + ar) * 8 + 2 * ak + 1] = make_double2(c1, c3);
      jt += P;
      __syncthreads();  // the group's ring slots are free, its partial tiles visible
      if (tid == 0)
        for (; ji < min(ntl, jt + TR); ++ji) issue_tile(ji);
      T.tick(3);
      if (own) {  // fixed-order sum over the warps that worked on this row tile
        const int t_o = orow >> 3, ro = orow & 7;
        for (int w2 = 0; w2 < P * KP; ++w2)
          if ((w2 % P) % nt == t_o) y = cadd(y, S.red[((w2 * IN_MG) * 8 + ro) * 8 + oq]);
      }
    }
    // ---- combine: t = y + (add0 + add1) - (sub0 + sub1); out = t | rev - t | t - rev
    if (own) {
      if (item.add[0].vec >= 0) y = cadd(y, addv);
      if (item.sub[0].vec >= 0) y = csub(y, subv);
      const int mode = item.flags >> 8 & 3;
      if (mode == 1) y = csub(revv, y);
      else if (mode == 2) y = csub(y, revv);
      vecp(p, job, rr, VM(item.dst.vec))[item.dst.seg * w + gi] = y;
    }
    __syncthreads();
    T.tick(4);
  }
  *tseq += (uint32_t)ntl;
}

// Execute one program (list of phases) for the active instances of this cluster.
// vmap: program vec ids {0:IN,1:OUT,2:AUX} -> scratch vector index.
__device__ void run_program(const InnerParams& p, int job, int layer, int w, int r0, const int* ph, int nph,
                            const int vmap[3], int nact, const InSmem& S, int q, int CS, uint32_t* tseq,
                            Ticker& T) {
  const int nmt = (w + 7) >> 3;
  const int MG = p.mg;  // 8-row tiles per group (shared-memory budget, from the widest layer)
  const int ngrp = (nmt + MG - 1) / MG;
  for (int phz = 0; phz < nph; ++phz) {
    const int it0 = ph[phz], nit = ph[phz + 1] - it0;
    // Weighted split of the phase's (item, tile group) pairs over the cluster: a pair weighs its
    // number of slot products (1 for a pure combination).  CTA q takes the pairs whose weight
    // midpoints fall in [q W / CS, (q+1) W / CS); a unit = (item, contiguous group range), its
    // panels gathered once.
    auto item_w = [&](int ii) { return S.items[it0 + ii].wgt; };
    int wtot = 0;
    for (int ii = 0; ii < nit; ++ii) wtot += item_w(ii) * ngrp;
    const int wlo2 = 2 * (int)((long long)q * wtot / CS), whi2 = 2 * (int)((long long)(q + 1) * wtot / CS);
    auto cdiv = [](int a, int b) { return a <= 0 ? -((-a) / b) : (a + b - 1) / b; };
    int wcum = 0;
    for (int ii = 0; ii < nit; ++ii) {
      const int wi = item_w(ii), wa = wcum;
      wcum += wi * ngrp;
      // group g's midpoint (doubled): 2 wa + wi (2g + 1)
      const int g0 = max(0, cdiv(wlo2 - 2 * wa - wi, 2 * wi));
      const int g1 = min(ngrp, cdiv(whi2 - 2 * wa - wi, 2 * wi));
      if (g0 >= g1) continue;
      T.tick(12);  // phase/unit bookkeeping
      const IItem& item = S.items[it0 + ii];
      item_unit(p, job, w, r0, S.act, nact, item, g0, g1, vmap, S, tseq, T, S.goff[item.cell >= 0 ? item.cell : 0]);
    }
    csync();
    T.tick(5);
  }
}

// y[inst][row] = sum_k M[row][k] x[inst][k] for the cluster's active instances, M row-major n x n: the dense
// inner operators (offline.py:inner_dense_operators).  DMMA m8n8k4 with the (up to 8) instances as N; CTA q
// takes row tiles [q T / CS, (q+1) T / CS) in chunks of DA_T, its 8 warps split the k-steps, and the partial
// tiles are summed in shared memory in a fixed warp order (deterministic).  Ends with a cluster barrier.
// y[inst][row] = sum_k M[row][k] x[inst][k] for the cluster's active instances: the dense inner operators
// (offline.py:inner_dense_operators), stored DMMA-fragment tile-major (k_dense_tiles).  CTA q takes the row
// tiles [q T / CS, (q+1) T / CS) in passes of up to DA_T tiles.  A pass streams, chunk by chunk (DA_KC k-steps),
// its tiles' fragments and the instances' x entries into a shared-memory ring with cp.async.bulk (thread 0
// produces, every warp releases each slot); warp wp takes k-step wp of each chunk and accumulates all the
// pass's tiles on DMMA (N = instances); the 8 warps' partial tiles are summed in a fixed order.  `dch` counts
// the chunks this CTA has streamed so far (ring phases persist across calls).  Ends with a cluster barrier.
#define DA_T 8
#define DA_NS 8
#define GV_MAX 32  // Arnoldi steps whose Givens state is staged in shared memory (beyond: global memory)
// One streaming pass over row tiles [t0, t1) of M for the instances rr[0..nact): see dense_apply.
// src < 0: x is rhs_pol gathered from the Newton tables (negated) instead of a scratch vector.
// ring/region: the shared-memory ring; dbar: DA_NS full + DA_NS empty barriers; the partial tiles reuse the
// ring.  A ring slot (fixed capacity dense_slot_bytes(scmax)) holds as many stored chunks (<= 16) of the pass's
// tiles as fit next to the instances' x entries for those k-steps, so passes over few tiles or few instances
// still move large slots.
__device__ __forceinline__ uint32_t dense_slot_bytes(int scmax) {
  return (uint32_t)DA_T * DA_KC * 512u + 8u * (uint32_t)(scmax * DA_KC * 4 + 4) * 16u;
}
__device__ void dense_pass(const InnerParams& p, const double2* __restrict__ Mt, int n, int job, const int* rr,
                           int nact, int src, int dst, int t0, int t1, unsigned char* ring, size_t region,
                           uint64_t* dbar, unsigned& dch, int scmax, int nmat = 1) {
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int ar = lane >> 2, ak = lane & 3;
  // nmat stacked matrices (row tiles of matrix m at [m T8m, (m+1) T8m)) share the pass's x: T8 = stored row
  // tiles per chunk, the output of stacked tile t goes to vector dst + t / T8m, row (t % T8m) * 8 + ar
  const int T8m = (n + 7) >> 3, T8 = nmat * T8m, nks = n >> 2;
  // fixed slot capacity (ring phases): the launcher's choice for the cooperative kernel, else by scmax
  const uint32_t slot_bytes = p.da_slot > 0 ? (uint32_t)p.da_slot : dense_slot_bytes(scmax);
  const int ns = (int)min((size_t)DA_NS, region / slot_bytes);
  uint64_t* full = dbar;
  uint64_t* empty = dbar + DA_NS;
  const int nchs = (nks + DA_KC - 1) / DA_KC;  // stored chunks
  for (int tc = t0; tc < t1; tc += DA_T) {
    const int nt = min(DA_T, t1 - tc);
    // stored chunks per slot: as many as the slot holds next to the instances' x rows (few tiles or few
    // instances -> more k per slot, more bytes in flight)
    int sc = 1;
    for (int cand = 16; cand > 1; --cand)
      if ((uint32_t)(cand * nt * DA_KC * 512 + nact * (cand * DA_KC * 4 + 4) * 16) <= slot_bytes) {
        sc = cand;
        break;
      }
    const int XST = sc * DA_KC * 4 + 4;                   // padded x row (double2) per instance
    const uint32_t abytes = (uint32_t)(sc * nt * DA_KC * 512);  // A part of this pass's slots
    const int kslot = sc * DA_KC;                  // k-steps per slot
    const int nsl = (nks + kslot - 1) / kslot;     // slots of this pass
    const unsigned base = dch;  // global index of this pass's slot 0
    // warp 0 fills slot c of this pass: lane 0 arms the barrier, lanes < nsub copy one stored chunk of the
    // pass's tiles each (contiguous in the chunk-major layout), lanes < nact copy instance x entries
    auto issue = [&](int c) {
      const unsigned g = base + (unsigned)c;
      const int sl = (int)(g % (unsigned)ns);
      const int k0 = c * kslot, kx = min(kslot, nks - k0);
      const int nsub = min(sc, nchs - c * sc);
      unsigned char* sp = ring + (size_t)sl * slot_bytes;
      if (lane == 0 && g >= (unsigned)ns) mbar_wait(&empty[sl], ((g / ns) - 1) & 1);
      __syncwarp();
      if (src < 0) {
        // x = rhs_pol gathered from the Newton tables (sie.py:230-242, negated) by the lanes of warp 0
        const int nIc = p.Lc - 1, w = n / (4 * nIc);
        double2* xs = reinterpret_cast<double2*>(sp + abytes);
        for (int ix = lane; ix < nact * kx * 4; ix += 32) {
          const int i = ix / (kx * 4), e = k0 * 4 + (ix - i * kx * 4);
          const int seg = e / w, j = e - seg * w;
          const int half = seg / (2 * nIc);  // 0 down, 1 up
          const int I = (seg % (2 * nIc)) / 2, s_ = seg & 1;
          const int cc = half == 0 ? I : I + 1;
          const int idx = half == 0 ? 2 + s_ : s_;
          const double2 tv = __ldcg(p.tables + ((((size_t)job * p.Lc + cc) * 4 + idx) * p.R + rr[i]) * p.wmax + j);
          xs[i * XST + (e - k0 * 4)] = make_double2(-tv.x, -tv.y);
        }
        // these generic stores precede later bulk copies into the same slot; published by the arrive below
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      }
      if (lane == 0)
        mbar_expect_tx(&full[sl], (uint32_t)(nsub * nt * DA_KC * 512 + (src >= 0 ? nact * kx * 64 : 0)));
      __syncwarp();
      if (lane < nsub)
        bulk_g2s(sp + (size_t)lane * nt * DA_KC * 512, Mt + ((size_t)(c * sc + lane) * T8 + tc) * DA_KC * 32,
                 (uint32_t)nt * DA_KC * 512u, &full[sl]);
      if (src >= 0 && lane < nact)
        bulk_g2s(sp + abytes + (size_t)lane * XST * 16, vecp(p, job, rr[lane], src) + (size_t)k0 * 4,
                 (uint32_t)kx * 64u, &full[sl]);
    };
    if (wp == 0)
      for (int c = 0; c < min(ns - 1, nsl); ++c) issue(c);
    double acc[DA_T][4];
#pragma unroll
    for (int t = 0; t < DA_T; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0;
    for (int c = 0; c < nsl; ++c) {
      if (wp == 0 && c + ns - 1 < nsl) issue(c + ns - 1);
      const unsigned g = base + (unsigned)c;
      const int sl = (int)(g % (unsigned)ns);
      const bool tw = p.tprof && blockIdx.x == 0 && tid == 32;  // warp 1: time spent waiting for data
      const long long tw0 = tw ? clock64() : 0;
      mbar_wait(&full[sl], (g / ns) & 1);
      if (tw) atomicAdd((unsigned long long*)&g_in_t[14], (unsigned long long)(clock64() - tw0));
      const int kx = min(kslot, nks - c * kslot);
      const unsigned char* sp = ring + (size_t)sl * slot_bytes;
      const double2* xs = reinterpret_cast<const double2*>(sp + abytes);
      // the tile count is a compile-time constant in each branch: no predicated-off DMMAs
#define DA_CONSUME(NT)                                                                                   \
  for (int kl = wp; kl < kx; kl += IN_THREADS / 32) {                                                    \
    const double2 bv = ar < nact ? xs[ar * XST + kl * 4 + ak] : czero();                                 \
    const int sub = kl / DA_KC, kk = kl - sub * DA_KC;                                                    \
    const double2* af = reinterpret_cast<const double2*>(sp) + ((size_t)sub * NT * DA_KC + kk) * 32 + lane; \
    _Pragma("unroll") for (int t = 0; t < NT; ++t) {                                                     \
      const double2 av = af[t * DA_KC * 32];                                                              \
      dmma_f64(acc[t][0], acc[t][1], av.x, bv.x);                                                         \
      dmma_f64(acc[t][2], acc[t][3], av.x, bv.y);                                                         \
      dmma_f64(acc[t][0], acc[t][1], -av.y, bv.y);                                                        \
      dmma_f64(acc[t][2], acc[t][3], av.y, bv.x);                                                         \
    }                                                                                                     \
  }
      switch (nt) {
        case 1: DA_CONSUME(1) break;
        case 2: DA_CONSUME(2) break;
        case 3: DA_CONSUME(3) break;
        case 4: DA_CONSUME(4) break;
        case 5: DA_CONSUME(5) break;
        case 6: DA_CONSUME(6) break;
        case 7: DA_CONSUME(7) break;
        default: DA_CONSUME(8) break;
      }
#undef DA_CONSUME
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
    }
    dch = base + (unsigned)nsl;
    __syncthreads();  // every slot consumed: the ring holds the partial tiles now
    double* part = reinterpret_cast<double*>(ring);  // [8 warps][DA_T][4][32]
#pragma unroll
    for (int t = 0; t < DA_T; ++t)
      if (t < nt)
#pragma unroll
        for (int v = 0; v < 4; ++v) part[((wp * DA_T + t) * 4 + v) * 32 + lane] = acc[t][v];
    __syncthreads();
    if (wp < nt) {  // warp wp owns tile tc + wp: fixed-order sum over the 8 k parts
      double c4[4] = {0.0, 0.0, 0.0, 0.0};
      for (int gw = 0; gw < IN_THREADS / 32; ++gw)
#pragma unroll
        for (int v = 0; v < 4; ++v) c4[v] += part[((gw * DA_T + wp) * 4 + v) * 32 + lane];
      const int ts = tc + wp, mi = ts / T8m;
      const int row = (ts - mi * T8m) * 8 + ar;
      if (row < n) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = 2 * ak + h;  // instance slot
          if (a < nact) vecp(p, job, rr[a], dst + mi)[row] = make_double2(c4[h], c4[2 + h]);
        }
      }
    }
    // the ring's generic-proxy use (partial tiles) must be ordered before the next bulk copies into it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
}

// Cluster version: CTA q of the cluster takes row tiles [q T / CS, (q+1) T / CS); ends with a cluster barrier.
__device__ void dense_apply(const InnerParams& p, const double2* __restrict__ Mt, int n, int job, int r0, int src,
                            int dst, int nact, const InSmem& S, int q, int CS, unsigned& dch) {
  const int T8 = (n + 7) >> 3;
  int rr[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) rr[i] = i < nact ? r0 + S.act[i] : r0;
  dense_pass(p, Mt, n, job, rr, nact, src, dst, q * T8 / CS, (q + 1) * T8 / CS, reinterpret_cast<unsigned char*>(S.tiles),
             S.region, S.dbar, dch, 1);
  csync();
}

// ---- per-instance GMRES steps (krylov.py:53-135), executed by the instance's owner CTA

// b = Y = pre(rhs): beta0 = ||b||, V_0 = b / beta0, Givens rhs g[0] = beta0, state
__device__ void instance_init(const InnerParams& p, int job, int r, int n, int VY, double* dred) {
  const int tid = threadIdx.x;
  const size_t hld = (size_t)p.cap + 1;
  const double2* Y = vecp(p, job, r, VY);
  double ss = 0.0;
  for (int e = tid; e < n; e += blockDim.x) {
    const double2 y = ld_cg(Y + e);
    ss += y.x * y.x + y.y * y.y;
  }
  ss = block_sum(ss, dred);
  const double b0 = sqrt(ss);
  double2* V0 = vecp(p, job, r, 0);
  if (b0 != 0.0) {
    const double ib0 = 1.0 / b0;
    for (int e = tid; e < n; e += blockDim.x) {
      const double2 y = ld_cg(Y + e);
      V0[e] = make_double2(y.x * ib0, y.y * ib0);
    }
  }
  if (tid == 0) {
    double2* g = p.hess + (size_t)(job * p.R + r) * p.hstride + hld * p.cap;
    g[0] = make_double2(b0, 0.0);
    p.beta0[job * p.R + r] = b0;
    p.state[job * p.R + r] = b0 == 0.0 ? 1 : 0;
    p.iters[job * p.R + r] = b0 == 0.0 ? 0 : -1;
  }
  __syncthreads();
}

// MGS Arnoldi + complex Givens for instance r at step j (krylov.py:89-127): W = V_{j+1} holds pre(op(V_j))
__device__ void instance_arnoldi(const InnerParams& p, int job, int r, int j, int n, double* dred,
                                 double wscale = 1.0) {
  const int tid = threadIdx.x;
  const size_t hld = (size_t)p.cap + 1;
  auto Hp = [&](int rr_) { return p.hess + (size_t)(job * p.R + rr_) * p.hstride; };
  double2* W = vecp(p, job, r, j + 1);
  double2* H = Hp(r);
  double2* col = H + (size_t)j * hld;
  // Givens state staged in shared memory: s_gv[0..j] = this column, s_gv[GV_MAX + i] = cs[i],
  // s_gv[2 GV_MAX + i] = sn[i]; the previous rotations and g[j] are loaded in parallel here, so the
  // serial rotation loop below runs on shared memory instead of dependent L2 round trips
  __shared__ double2 s_gv[3 * GV_MAX + 2];
  __shared__ double s_b0;
  const bool gsm = j + 2 <= GV_MAX;
  if (gsm) {
    const double2* gg = H + hld * p.cap;
    const double2* css = gg + (p.cap + 1);
    const double2* snn = css + p.cap;
    for (int i = tid; i < j; i += blockDim.x) {
      s_gv[GV_MAX + i] = css[i];
      s_gv[2 * GV_MAX + i] = snn[i];
    }
    if (tid == 0) {
      s_gv[3 * GV_MAX] = gg[j];
      s_b0 = p.beta0[job * p.R + r];
    }
  }
  double ss = 0.0;
  constexpr int EPT = 8;  // register-resident w for n <= EPT * IN_THREADS
  constexpr int FE = 4, FV = 6;  // fast path: n <= FE * IN_THREADS, j < FV (every V_i prefetched)
  double2 fw[FE];
  const bool fast = p.arn_fast && gsm && n <= FE * IN_THREADS && j < FV;
  if (fast) {
    // W and every V_i (i <= j) issued before the first reduction: one L2 round trip instead of j + 3; the
    // same per-thread element order and block sums as the path below (bitwise identical results)
    double2 fv[FV][FE];
#pragma unroll
    for (int t = 0; t < FE; ++t) {
      const int e = tid + t * IN_THREADS;
      fw[t] = e < n ? ld_cg(W + e) : czero();
      fw[t].x *= wscale;
      fw[t].y *= wscale;
    }
#pragma unroll
    for (int i = 0; i < FV; ++i)
      if (i <= j) {
        const double2* Vi = vecp(p, job, r, i);
#pragma unroll
        for (int t = 0; t < FE; ++t) {
          const int e = tid + t * IN_THREADS;
          fv[i][t] = e < n ? ld_cg(Vi + e) : czero();
        }
      }
#pragma unroll
    for (int i = 0; i < FV; ++i) {
      if (i > j) break;
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int t = 0; t < FE; ++t) {
        const double2 c = cconjmul(fv[i][t], fw[t]);
        sr += c.x;
        si += c.y;
      }
      const double2 h = block_sum2(sr, si, dred);
      if (tid == 0) {
        col[i] = h;
        s_gv[i] = h;
      }
#pragma unroll
      for (int t = 0; t < FE; ++t) fw[t] = csub(fw[t], cmul(h, fv[i][t]));
    }
#pragma unroll
    for (int t = 0; t < FE; ++t) ss += fw[t].x * fw[t].x + fw[t].y * fw[t].y;
  } else if (n <= EPT * IN_THREADS) {
    double2 wv[EPT];
#pragma unroll
    for (int t = 0; t < EPT; ++t) {
      const int e = tid + t * IN_THREADS;
      wv[t] = e < n ? ld_cg(W + e) : czero();
      wv[t].x *= wscale;
      wv[t].y *= wscale;
    }
    for (int i = 0; i <= j; ++i) {
      const double2* Vi = vecp(p, job, r, i);
      double2 vv[EPT];
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int t = 0; t < EPT; ++t) {
        const int e = tid + t * IN_THREADS;
        vv[t] = e < n ? ld_cg(Vi + e) : czero();
        const double2 c = cconjmul(vv[t], wv[t]);
        sr += c.x;
        si += c.y;
      }
      const double2 h = block_sum2(sr, si, dred);
      if (tid == 0) {
        col[i] = h;
        if (i < GV_MAX) s_gv[i] = h;
      }
#pragma unroll
      for (int t = 0; t < EPT; ++t) wv[t] = csub(wv[t], cmul(h, vv[t]));
    }
#pragma unroll
    for (int t = 0; t < EPT; ++t) {
      const int e = tid + t * IN_THREADS;
      if (e < n) W[e] = wv[t];
      ss += wv[t].x * wv[t].x + wv[t].y * wv[t].y;
    }
  } else {
    if (wscale != 1.0) {
      for (int e = tid; e < n; e += blockDim.x) {
        const double2 x = ld_cg(W + e);
        W[e] = make_double2(x.x * wscale, x.y * wscale);
      }
      __syncthreads();
    }
    for (int i = 0; i <= j; ++i) {
      const double2* Vi = vecp(p, job, r, i);
      double sr = 0.0, si = 0.0;
      for (int e = tid; e < n; e += blockDim.x) {
        const double2 c = cconjmul(ld_cg(Vi + e), ld_cg(W + e));
        sr += c.x;
        si += c.y;
      }
      const double2 h = block_sum2(sr, si, dred);
      if (tid == 0) {
        col[i] = h;
        if (i < GV_MAX) s_gv[i] = h;
      }
      for (int e = tid; e < n; e += blockDim.x) W[e] = csub(ld_cg(W + e), cmul(h, ld_cg(Vi + e)));
      __syncthreads();
    }
    for (int e = tid; e < n; e += blockDim.x) {
      const double2 x = W[e];
      ss += x.x * x.x + x.y * x.y;
    }
  }
  ss = block_sum(ss, dred);
  const double hn = sqrt(ss);
  __shared__ int s_st;
  if (tid == 0 && gsm) {  // rotations on shared memory, results written back to the global Hessenberg
    double2* g = H + hld * p.cap;
    double2* cs = g + (p.cap + 1);
    double2* sn = cs + p.cap;
    double2* cl = s_gv;
    cl[j + 1] = make_double2(hn, 0.0);
    for (int i = 0; i < j; ++i) {
      const double2 csi = s_gv[GV_MAX + i], sni = s_gv[2 * GV_MAX + i];
      const double2 t = cadd(cmul(csi, cl[i]), cmul(sni, cl[i + 1]));
      const double2 nsc = make_double2(-sni.x, sni.y);  // -conj(sn)
      const double2 csc = make_double2(csi.x, -csi.y);  // conj(cs)
      cl[i + 1] = cadd(cmul(nsc, cl[i]), cmul(csc, cl[i + 1]));
      cl[i] = t;
    }
    const double aa = hypot(cl[j].x, cl[j].y);
    const double d = sqrt(aa * aa + hn * hn);
    int st = 0;  // 0 continue, 1 converged, 2 failed
    if (d == 0.0) {
      st = 2;
      atomicMax(p.err, 3);
    } else {
      const double2 c = make_double2(cl[j].x / d, -cl[j].y / d);
      const double2 sv = make_double2(hn / d, 0.0);
      cs[j] = c;
      sn[j] = sv;
      cl[j] = cadd(cmul(c, cl[j]), make_double2(sv.x * hn, 0.0));
      const double2 gj = s_gv[3 * GV_MAX];
      const double2 gj1 = cmul(make_double2(-sv.x, sv.y), gj);
      g[j + 1] = gj1;
      g[j] = cmul(c, gj);
      const double res = hypot(gj1.x, gj1.y) / s_b0;
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
    for (int i = 0; i <= j + 1; ++i) col[i] = cl[i];
    s_st = st;
    p.state[job * p.R + r] = st;
    if (st != 0) p.iters[job * p.R + r] = st == 1 ? j + 1 : -1;
  }
  if (tid == 0 && !gsm) {
    double2* g = H + hld * p.cap;
    double2* cs = g + (p.cap + 1);
    double2* sn = cs + p.cap;
    col[j + 1] = make_double2(hn, 0.0);
    for (int i = 0; i < j; ++i) {
      const double2 t = cadd(cmul(cs[i], col[i]), cmul(sn[i], col[i + 1]));
      const double2 nsc = make_double2(-sn[i].x, sn[i].y);  // -conj(sn)
      const double2 csc = make_double2(cs[i].x, -cs[i].y);  // conj(cs)
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
      const double2 s = make_double2(hn / d, 0.0);
      cs[j] = c;
      sn[j] = s;
      col[j] = cadd(cmul(c, col[j]), make_double2(s.x * hn, 0.0));
      const double2 gj = g[j];
      g[j + 1] = cmul(make_double2(-s.x, s.y), gj);
      g[j] = cmul(c, gj);
      const double res = hypot(g[j + 1].x, g[j + 1].y) / p.beta0[job * p.R + r];
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
    s_st = st;
    p.state[job * p.R + r] = st;
    if (st != 0) p.iters[job * p.R + r] = st == 1 ? j + 1 : -1;
  }
  __syncthreads();
  const double ihn = 1.0 / hn;  // scalings as products with the reciprocal (FP64 division is slow)
  if (fast) {  // V_{j+1} = w / hn from registers (the orthogonalized w itself once the instance stops)
#pragma unroll
    for (int t = 0; t < FE; ++t) {
      const int e = tid + t * IN_THREADS;
      if (e < n) W[e] = s_st == 0 ? make_double2(fw[t].x * ihn, fw[t].y * ihn) : fw[t];
    }
  } else if (s_st == 0) {  // V_{j+1} = w / hn (krylov.py:125)
    for (int e = tid; e < n; e += blockDim.x) {
      const double2 x = W[e];
      W[e] = make_double2(x.x * ihn, x.y * ihn);
    }
  }
  __syncthreads();
}

// One Givens step of krylov.py:97-127 on thread 0 with the rotation state in registers (no global read-back):
// column col[0..j+1] (col[j+1] = hn on entry), rotations cs/sn[0..j), g[0..j] of instance (job, r) and its
// beta0 b0.  Forms rotation j, updates g, writes the column, the rotation, g and the state / iteration count as
// instance_arnoldi does.  Returns the state (0 running, 1 converged, 2 failed).
__device__ int givens_col(const InnerParams& p, int job, int r, int j, double2* col, double hn, double2* cs,
                          double2* sn, double2* g, double b0) {
  const size_t hld = (size_t)p.cap + 1;
  double2* H = p.hess + (size_t)(job * p.R + r) * p.hstride;
  double2* gG = H + hld * p.cap;
  double2* csG = gG + (p.cap + 1);
  double2* snG = csG + p.cap;
  for (int i = 0; i < j; ++i) {
    const double2 t = cadd(cmul(cs[i], col[i]), cmul(sn[i], col[i + 1]));
    const double2 nsc = make_double2(-sn[i].x, sn[i].y);  // -conj(sn)
    const double2 csc = make_double2(cs[i].x, -cs[i].y);  // conj(cs)
    col[i + 1] = cadd(cmul(nsc, col[i]), cmul(csc, col[i + 1]));
    col[i] = t;
  }
  const double aa = hypot(col[j].x, col[j].y);
  const double d = sqrt(aa * aa + hn * hn);
  int st = 0;
  if (d == 0.0) {
    st = 2;
    atomicMax(p.err, 3);
  } else {
    const double2 c = make_double2(col[j].x / d, -col[j].y / d);
    const double2 sv = make_double2(hn / d, 0.0);
    cs[j] = c;
    sn[j] = sv;
    csG[j] = c;
    snG[j] = sv;
    col[j] = cadd(cmul(c, col[j]), make_double2(sv.x * hn, 0.0));
    const double2 gj = g[j];
    const double2 gj1 = cmul(make_double2(-sv.x, sv.y), gj);
    g[j + 1] = gj1;
    g[j] = cmul(c, gj);
    gG[j + 1] = gj1;
    gG[j] = g[j];
    const double res = hypot(gj1.x, gj1.y) / b0;
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
  double2* hc = H + (size_t)j * hld;
  for (int i = 0; i <= j + 1; ++i) hc[i] = col[i];
  p.state[job * p.R + r] = st;
  if (st != 0) p.iters[job * p.R + r] = st == 1 ? j + 1 : -1;
  return st;
}

// instance_final for an instance that stopped inside the register s-step (k = 1 or 2): the basis vectors are
// still in registers (v0, v1), the triangle and g on thread 0's shared copies.  Same back substitution, x = V y
// order and accounting as instance_final; the halves of x meet through the shared scratch xs (>= n double2).
// Marks the instance finalized (state 3: stopped, traces written).
template <int SE>
__device__ void sstep_final(const InnerParams& p, int job, int r, int n, int k, const double2 (&v0)[SE],
                            const double2 (&v1)[SE], const double2* rtri, const double2* gk, double2* xs) {
  const int tid = threadIdx.x, nIc = p.Lc - 1, w = n / (4 * nIc);
  __shared__ double2 s_y[2];
  if (tid == 0) {  // rtri = (R00, R01, R11)
    double2 y[2] = {czero(), czero()};
    for (int i = k - 1; i >= 0; --i) {
      double2 sacc = czero();
      if (i == 0 && k == 2) cfma(sacc, rtri[1], y[1]);
      const double2 num = csub(gk[i], sacc);
      const double2 den = i == 0 ? rtri[0] : rtri[2];
      const double dd = den.x * den.x + den.y * den.y;
      y[i] = make_double2((num.x * den.x + num.y * den.y) / dd, (num.y * den.x - num.x * den.y) / dd);
    }
    s_y[0] = y[0];
    s_y[1] = y[1];
  }
  __syncthreads();
  const double2 y0 = s_y[0], y1 = s_y[1];
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    const int e = tid + t * IN_THREADS;
    if (e < n) {
      double2 x = czero();
      cfma(x, v0[t], y0);
      if (k == 2) cfma(x, v1[t], y1);
      xs[e] = x;
    }
  }
  __syncthreads();
  const int half = n / 2;
  double2* out = p.tr + (size_t)(job * p.R + r) * nIc * 2 * p.wmax;
  for (int e = tid; e < half; e += IN_THREADS) {
    const int seg = e / w, jj = e - seg * w;
    out[(size_t)seg * p.wmax + jj] = cadd(xs[e], xs[e + half]);
  }
  if (tid == 0) {  // TouchCounter.total equivalent (nested.py:54-73), as instance_final
    atomicAdd(&p.hist[min(k, PT_HIST - 1)], 1);
    atomicAdd(&p.counters[0], (unsigned long long)k);
    const unsigned long long t =
        ((unsigned long long)(k + 1) * p.pre_blocks + (unsigned long long)k * p.op_blocks) * w * w;
    atomicAdd(&p.counters[1], t);
    atomicAdd(&p.counters[2], 1ULL);
    p.state[job * p.R + r] = 3;
  }
  // xs is the dense ring: order these generic writes before later bulk copies into it
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
}

// s-step start of the inner GMRES (krylov.py:61-127, steps j = 0 and 1) for one instance, from m0 = b = pre(rhs)
// (VY), m1 = E b (VT) and m2 = E^2 b (VA), E = pre(op(.)) - I, all three produced by ONE dense pass: A V = E V + V
// gives the two products of the Arnoldi steps without waiting for the GPU in between.  The MGS, norms, Givens
// rotations and state are krylov.py's; only A V_j is formed from the shifted powers instead of a fresh product.
// Leaves V_0..V_2 (as far as the instance runs), H columns 0-1 and the Givens state as instance_arnoldi would.
// n <= SE * IN_THREADS.
__device__ void instance_sstep(const InnerParams& p, int job, int r, int n, int VY, int VT, int VA,
                               double* dred, double2* xs) {
  constexpr int SE = 4;
  const int tid = threadIdx.x;
  const double2* M0 = vecp(p, job, r, VY);
  const double2* M1 = vecp(p, job, r, VT);
  const double2* M2 = vecp(p, job, r, VA);
  double2 m0[SE], m1[SE], m2[SE], w[SE], v1[SE];
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    const int e = tid + t * IN_THREADS;
    m0[t] = e < n ? ld_cg(M0 + e) : czero();
    m1[t] = e < n ? ld_cg(M1 + e) : czero();
    m2[t] = e < n ? ld_cg(M2 + e) : czero();
  }
  __shared__ double2 s_col[4];
  __shared__ double2 s_tri[3];  // R00, R01, R11 of the triangularized Hessenberg (thread 0)
  __shared__ int s_st;
  // beta0 = ||b|| (instance_init)
  double ss = 0.0;
#pragma unroll
  for (int t = 0; t < SE; ++t) ss += m0[t].x * m0[t].x + m0[t].y * m0[t].y;
  ss = block_sum(ss, dred);
  const double b0 = sqrt(ss);
  const bool tp_on = p.tprof && tid == 0 && blockIdx.x == 0;
  long long tp0 = tp_on ? clock64() : 0;
  if (tid == 0) {
    double2* g = p.hess + (size_t)(job * p.R + r) * p.hstride + ((size_t)p.cap + 1) * p.cap;
    g[0] = make_double2(b0, 0.0);
    p.beta0[job * p.R + r] = b0;
    p.state[job * p.R + r] = b0 == 0.0 ? 1 : 0;
    p.iters[job * p.R + r] = b0 == 0.0 ? 0 : -1;
  }
  if (b0 == 0.0) {  // converged with zero iterations (krylov.py:62-65)
    __syncthreads();
    return;
  }
  double2* V0 = vecp(p, job, r, 0);
  // ---- j = 0: V_0 = b / beta0, w = A V_0 = E b / beta0 + V_0 (scalings as products with the reciprocal)
  const double ib0 = 1.0 / b0;
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    const int e = tid + t * IN_THREADS;
    const double2 v0 = make_double2(m0[t].x * ib0, m0[t].y * ib0);
    m0[t] = v0;                                             // m0 holds V_0 from here
    m1[t] = make_double2(m1[t].x * ib0, m1[t].y * ib0);     // E V_0
    m2[t] = make_double2(m2[t].x * ib0, m2[t].y * ib0);     // E^2 V_0
    if (e < n) V0[e] = v0;
    w[t] = cadd(m1[t], v0);
  }
  double sr = 0.0, si = 0.0;
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    const double2 c = cconjmul(m0[t], w[t]);
    sr += c.x;
    si += c.y;
  }
  const double2 h00 = block_sum2(sr, si, dred);
  ss = 0.0;
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    w[t] = csub(w[t], cmul(h00, m0[t]));
    ss += w[t].x * w[t].x + w[t].y * w[t].y;
  }
  const double hn0 = sqrt(block_sum(ss, dred));
  __shared__ double2 s_rot[7];  // cs[0..1], sn[0..1], g[0..2] of the Givens process (thread 0)
  if (tid == 0) {
    s_rot[4] = make_double2(b0, 0.0);  // g[0] = beta0
    s_col[0] = h00;
    s_col[1] = make_double2(hn0, 0.0);
    s_st = givens_col(p, job, r, 0, s_col, hn0, s_rot, s_rot + 2, s_rot + 4, b0);
    s_tri[0] = s_col[0];  // R00
  }
  __syncthreads();
  if (tp_on) {
    const long long t1 = clock64();
    atomicAdd((unsigned long long*)&g_in_t[0], (unsigned long long)(t1 - tp0));
    tp0 = t1;
  }
  if (s_st == 1 && xs) sstep_final<SE>(p, job, r, n, 1, m0, m0, s_tri, s_rot + 4, xs);
  if (s_st != 0) return;
  // ---- j = 1: V_1 = w / hn0, E V_1 = (E^2 V_0 + E V_0 - h00 E V_0) / hn0, w = E V_1 + V_1
  double2* V1 = vecp(p, job, r, 1);
  const double ihn0 = 1.0 / hn0;
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    const int e = tid + t * IN_THREADS;
    v1[t] = make_double2(w[t].x * ihn0, w[t].y * ihn0);
    if (e < n) V1[e] = v1[t];
    const double2 ev = csub(cadd(m2[t], m1[t]), cmul(h00, m1[t]));
    w[t] = cadd(make_double2(ev.x * ihn0, ev.y * ihn0), v1[t]);
  }
  sr = si = 0.0;
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    const double2 c = cconjmul(m0[t], w[t]);
    sr += c.x;
    si += c.y;
  }
  const double2 h01 = block_sum2(sr, si, dred);
  sr = si = 0.0;
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    w[t] = csub(w[t], cmul(h01, m0[t]));
    const double2 c = cconjmul(v1[t], w[t]);
    sr += c.x;
    si += c.y;
  }
  const double2 h11 = block_sum2(sr, si, dred);
  ss = 0.0;
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    w[t] = csub(w[t], cmul(h11, v1[t]));
    ss += w[t].x * w[t].x + w[t].y * w[t].y;
  }
  const double hn1 = sqrt(block_sum(ss, dred));
  if (tid == 0) {
    s_col[0] = h01;
    s_col[1] = h11;
    s_col[2] = make_double2(hn1, 0.0);
    s_st = givens_col(p, job, r, 1, s_col, hn1, s_rot, s_rot + 2, s_rot + 4, b0);
    s_tri[1] = s_col[0];  // R01
    s_tri[2] = s_col[1];  // R11
  }
  __syncthreads();
  if (tp_on) atomicAdd((unsigned long long*)&g_in_t[1], (unsigned long long)(clock64() - tp0));
  if (s_st == 1 && xs) sstep_final<SE>(p, job, r, n, 2, m0, v1, s_tri, s_rot + 4, xs);
  if (s_st != 0) return;
  double2* V2 = vecp(p, job, r, 2);  // V_2 = w / hn1: the regular loop continues at j = 2
  const double ihn1 = 1.0 / hn1;
#pragma unroll
  for (int t = 0; t < SE; ++t) {
    const int e = tid + t * IN_THREADS;
    if (e < n) V2[e] = make_double2(w[t].x * ihn1, w[t].y * ihn1);
  }
  __syncthreads();
}

// instance_sstep for any n: the same quantities, every pass recomputed elementwise from m0, m1, m2 (read from
// L2) instead of held in registers.  Element e belongs to thread e % IN_THREADS; each reduction sums a thread's
// elements in increasing e, then block_sum in warp order (deterministic).
__device__ void instance_sstep_loop(const InnerParams& p, int job, int r, int n, int VY, int VT, int VA,
                                    double* dred) {
  const int tid = threadIdx.x;
  const double2* M0 = vecp(p, job, r, VY);
  const double2* M1 = vecp(p, job, r, VT);
  const double2* M2 = vecp(p, job, r, VA);
  __shared__ double2 s_col[4];
  __shared__ double2 s_rot[7];
  __shared__ int s_st;
  double ss = 0.0;
  for (int e = tid; e < n; e += IN_THREADS) {
    const double2 a = ld_cg(M0 + e);
    ss += a.x * a.x + a.y * a.y;
  }
  const double b0 = sqrt(block_sum(ss, dred));
  if (tid == 0) {
    double2* g = p.hess + (size_t)(job * p.R + r) * p.hstride + ((size_t)p.cap + 1) * p.cap;
    g[0] = make_double2(b0, 0.0);
    p.beta0[job * p.R + r] = b0;
    p.state[job * p.R + r] = b0 == 0.0 ? 1 : 0;
    p.iters[job * p.R + r] = b0 == 0.0 ? 0 : -1;
  }
  if (b0 == 0.0) {
    __syncthreads();
    return;
  }
  double2* V0 = vecp(p, job, r, 0);
  double2* V1 = vecp(p, job, r, 1);
  double2* V2 = vecp(p, job, r, 2);
  const double ib0 = 1.0 / b0;
  auto sc = [](double2 a, double d) { return make_double2(a.x * d, a.y * d); };  // d: a reciprocal
  // ---- j = 0: V_0 = m0 / b0, w = E V_0 + V_0
  double sr = 0.0, si = 0.0;
  for (int e = tid; e < n; e += IN_THREADS) {
    const double2 v0 = sc(ld_cg(M0 + e), ib0);
    V0[e] = v0;
    const double2 c = cconjmul(v0, cadd(sc(ld_cg(M1 + e), ib0), v0));
    sr += c.x;
    si += c.y;
  }
  const double2 h00 = block_sum2(sr, si, dred);
  ss = 0.0;
  for (int e = tid; e < n; e += IN_THREADS) {
    const double2 v0 = sc(ld_cg(M0 + e), ib0);
    const double2 w = csub(cadd(sc(ld_cg(M1 + e), ib0), v0), cmul(h00, v0));
    ss += w.x * w.x + w.y * w.y;
  }
  const double hn0 = sqrt(block_sum(ss, dred));
  if (tid == 0) {
    s_rot[4] = make_double2(b0, 0.0);
    s_col[0] = h00;
    s_col[1] = make_double2(hn0, 0.0);
    s_st = givens_col(p, job, r, 0, s_col, hn0, s_rot, s_rot + 2, s_rot + 4, b0);
  }
  __syncthreads();
  if (s_st != 0) return;
  // ---- j = 1: V_1 = w / hn0, E V_1 = (E^2 V_0 + E V_0 - h00 E V_0) / hn0, w = E V_1 + V_1
  const double ihn0 = 1.0 / hn0;
  auto v1_of = [&](int e, double2& v0, double2& v1, double2& w1) {
    v0 = sc(ld_cg(M0 + e), ib0);
    const double2 e0 = sc(ld_cg(M1 + e), ib0);
    v1 = sc(csub(cadd(e0, v0), cmul(h00, v0)), ihn0);
    const double2 ev = csub(cadd(sc(ld_cg(M2 + e), ib0), e0), cmul(h00, e0));
    w1 = cadd(sc(ev, ihn0), v1);
  };
  sr = si = 0.0;
  for (int e = tid; e < n; e += IN_THREADS) {
    double2 v0, v1, w1;
    v1_of(e, v0, v1, w1);
    V1[e] = v1;
    const double2 c = cconjmul(v0, w1);
    sr += c.x;
    si += c.y;
  }
  const double2 h01 = block_sum2(sr, si, dred);
  sr = si = 0.0;
  for (int e = tid; e < n; e += IN_THREADS) {
    double2 v0, v1, w1;
    v1_of(e, v0, v1, w1);
    const double2 c = cconjmul(v1, csub(w1, cmul(h01, v0)));
    sr += c.x;
    si += c.y;
  }
  const double2 h11 = block_sum2(sr, si, dred);
  ss = 0.0;
  for (int e = tid; e < n; e += IN_THREADS) {
    double2 v0, v1, w1;
    v1_of(e, v0, v1, w1);
    const double2 w = csub(csub(w1, cmul(h01, v0)), cmul(h11, v1));
    ss += w.x * w.x + w.y * w.y;
  }
  const double hn1 = sqrt(block_sum(ss, dred));
  if (tid == 0) {
    s_col[0] = h01;
    s_col[1] = h11;
    s_col[2] = make_double2(hn1, 0.0);
    s_st = givens_col(p, job, r, 1, s_col, hn1, s_rot, s_rot + 2, s_rot + 4, b0);
  }
  __syncthreads();
  if (s_st != 0) return;
  const double ihn1 = 1.0 / hn1;
  for (int e = tid; e < n; e += IN_THREADS) {
    double2 v0, v1, w1;
    v1_of(e, v0, v1, w1);
    V2[e] = sc(csub(csub(w1, cmul(h01, v0)), cmul(h11, v1)), ihn1);
  }
  __syncthreads();
}

// b = Y = pre(rhs) and W = V_1 = pre(op(b)) (the product taken on the unnormalized b): beta0 = ||b||,
// V_0 = b / beta0, then the Arnoldi step j = 0 on W / beta0 (= pre(op(V_0)) up to rounding)
__device__ void instance_arnoldi0(const InnerParams& p, int job, int r, int n, int VY, double* dred) {
  instance_init(p, job, r, n, VY, dred);
  __shared__ double s_b0i;
  if (threadIdx.x == 0) s_b0i = p.beta0[job * p.R + r];
  __syncthreads();
  const double b0 = s_b0i;
  if (b0 == 0.0) return;  // converged with zero iterations (krylov.py:62-65)
  instance_arnoldi(p, job, r, 0, n, dred, 1.0 / b0);
}

// x = V_k y (back substitution on the triangularized Hessenberg), traces = down + up (nested.py:153),
// TouchCounter accounting (nested.py:54-73); yv: shared scratch of >= cap double2
__device__ void instance_final(const InnerParams& p, int job, int r, int n, int w, double2* yv) {
  const int tid = threadIdx.x;
  const int nIc = p.Lc - 1;
  const size_t hld = (size_t)p.cap + 1;
  auto Hp = [&](int rr_) { return p.hess + (size_t)(job * p.R + rr_) * p.hstride; };
  __shared__ int s_k;
  if (tid == 0) s_k = p.iters[job * p.R + r];
  __syncthreads();
  const int k = s_k;
  // the upper triangle H[0..k)[0..k) and g[0..k) staged in shared memory by all threads (k <= 24: 300
  // entries after yv), then the back substitution runs on thread 0 without dependent L2 round trips
  constexpr int KS = 24;
  double2* hs = yv + KS;  // [k(k+1)/2] column m holds rows 0..m
  double2* gs = hs + KS * (KS + 1) / 2;
  const double2* H = Hp(r);
  const double2* g = H + hld * p.cap;
  if (k > 0 && k <= KS) {
    for (int e = tid; e < k * (k + 1) / 2; e += blockDim.x) {
      int m = 0;
      while ((m + 1) * (m + 2) / 2 <= e) ++m;
      const int i = e - m * (m + 1) / 2;
      hs[e] = H[(size_t)m * hld + i];
    }
    for (int i = tid; i < k; i += blockDim.x) gs[i] = g[i];
  }
  __syncthreads();
  if (tid == 0 && k > 0) {
    const bool sm = k <= KS;
    for (int i = k - 1; i >= 0; --i) {
      double2 s = czero();
      for (int m = i + 1; m < k; ++m) cfma(s, sm ? hs[m * (m + 1) / 2 + i] : H[(size_t)m * hld + i], yv[m]);
      const double2 num = csub(sm ? gs[i] : g[i], s);
      const double2 den = sm ? hs[i * (i + 1) / 2 + i] : H[(size_t)i * hld + i];
      const double dd = den.x * den.x + den.y * den.y;
      yv[i] = make_double2((num.x * den.x + num.y * den.y) / dd, (num.y * den.x - num.x * den.y) / dd);
    }
  }
  __syncthreads();
  const int half = n / 2;
  double2* out = p.tr + (size_t)(job * p.R + r) * nIc * 2 * p.wmax;
  for (int e = tid; e < half; e += blockDim.x) {
    double2 xd = czero(), xu = czero();
    for (int i = 0; i < k; ++i) {
      const double2* Vi = vecp(p, job, r, i);
      cfma(xd, ld_cg(Vi + e), yv[i]);
      cfma(xu, ld_cg(Vi + half + e), yv[i]);
    }
    const int seg = e / w, jj = e - seg * w;
    out[(size_t)seg * p.wmax + jj] = cadd(xd, xu);
  }
  // ---- accounting: TouchCounter.total equivalent (nested.py:54-73)
  if (tid == 0 && k >= 0) {
    atomicAdd(&p.hist[min(k, PT_HIST - 1)], 1);
    atomicAdd(&p.counters[0], (unsigned long long)k);
    const unsigned long long t =
        ((unsigned long long)(k + 1) * p.pre_blocks + (unsigned long long)k * p.op_blocks) * w * w;
    atomicAdd(&p.counters[1], t);
    atomicAdd(&p.counters[2], 1ULL);
  }
  __syncthreads();
}

// rebuild the (cluster-consistent) list of active local instances from global state
__device__ __forceinline__ void rebuild_active(const InnerParams& p, int job, int r0, int ni, int* act, int* s_nact) {
  if (threadIdx.x == 0) {
    int na = 0;
    for (int l = 0; l < ni; ++l)
      if (__ldcg(p.state + job * p.R + r0 + l) == 0) act[na++] = l;
    *s_nact = na;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(IN_THREADS, 1)
    inner_gmres_kernel(const InnerParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int CS = (int)cg::this_cluster().num_blocks();  // 8 or 16 (launch attribute)
  const int q = (int)cg::this_cluster().block_rank();
  const int ngroups = (p.R + 7) >> 3;
  const int cid = blockIdx.x / CS;
  const int job = p.stage_jobs[cid / ngroups];
  const int r0 = (cid % ngroups) * 8;
  const int ni = min(8, p.R - r0);  // instances of this cluster: r0 .. r0+ni-1
  const int layer = p.jobs[job].layer;
  const int w = p.layers[layer].w;
  const int nIc = p.Lc - 1;
  const int n = 4 * nIc * w;
  const int tid = threadIdx.x;
  const long long tk_entry = clock64();

  InSmem S;
  S.tiles = reinterpret_cast<double2*>(smem);
  S.pan = S.tiles + (size_t)p.tring * p.wmax * 8;
  S.pan2 = S.pan + (size_t)4 * p.wmax * 8;
  S.red = S.pan2 + (size_t)2 * p.wmax * 8;
  double* dred = reinterpret_cast<double*>(S.red + (IN_THREADS / 32) * IN_MG * 8 * 8);
  S.tbar = reinterpret_cast<uint64_t*>(dred + 64);
  S.region = (size_t)(reinterpret_cast<unsigned char*>(dred) - reinterpret_cast<unsigned char*>(S.tiles));
  S.dbar = S.tbar + IN_TRMAX;
  S.act = reinterpret_cast<int*>(S.dbar + 2 * DA_NS);
  S.goff = reinterpret_cast<long long*>(S.act + 16);
  S.oph = reinterpret_cast<int*>(S.goff + PT_MAX_LC);
  S.pph = S.oph + 2 * PT_MAX_LC + 2;
  S.items = reinterpret_cast<IItem*>(S.pph + 2 * PT_MAX_LC + 2);
  __shared__ int s_nact;
  if (nIc == 0) return;
  if (tid == 0) {
    for (int i = 0; i < IN_TRMAX; ++i) mbar_init(&S.tbar[i], 1);
    for (int i = 0; i < DA_NS; ++i) {
      mbar_init(&S.dbar[i], 1);
      mbar_init(&S.dbar[DA_NS + i], IN_THREADS / 32);
    }
    fence_mbar_init();
  }
  for (int i = tid; i < p.nitems; i += blockDim.x) S.items[i] = p.items[i];
  for (int i = tid; i <= p.op_nph; i += blockDim.x) S.oph[i] = p.op_ph[i];
  for (int i = tid; i <= p.pre_nph; i += blockDim.x) S.pph[i] = p.pre_ph[i];
  for (int i = tid; i < p.Lc; i += blockDim.x) S.goff[i] = p.cells[layer * p.Lc + i].green_off;
  uint32_t tseq = 0;
  Ticker T;
  T.on = p.tprof && blockIdx.x == 0 && tid == 0;
  T.start();
  const int VB = p.cap + 1, VY = p.cap + 2, VT = p.cap + 3, VA = p.cap + 4;

  // ---- rhs_pol from the Newton tables (sie.py:230-242, negated); elements split over the cluster
  for (int l = 0; l < ni; ++l) {
    const int r = r0 + l;
    double2* B = vecp(p, job, r, VB);
    for (int e = q * blockDim.x + tid; e < n; e += CS * blockDim.x) {
      const int seg = e / w, j = e - seg * w;
      const int half = seg / (2 * nIc);  // 0 down, 1 up
      const int I = (seg % (2 * nIc)) / 2, s = seg & 1;
      const int c = half == 0 ? I : I + 1;
      const int idx = half == 0 ? 2 + s : s;  // down: rn, rnp of cell I; up: r0, r1 of cell I+1
      const double2 t = __ldcg(p.tables + ((((size_t)job * p.Lc + c) * 4 + idx) * p.R + r) * p.wmax + j);
      B[e] = make_double2(-t.x, -t.y);
    }
  }
  if (tid < ni) S.act[tid] = tid;
  if (tid == 0) s_nact = ni;
  csync();
  T.tick(8);

  // dense inner operators [pre; pre o op] of this layer, if provided
  const long long doff = p.layers[layer].dense_off;
  // the dense path needs two ring slots (DA_T tiles x DA_KC k-steps + 8 x-rows) and the partial tiles
  const bool dense_ok = S.region >= 2 * ((size_t)DA_T * DA_KC * 512 + 8 * (DA_KC * 4 + 4) * 16) &&
                        S.region >= (size_t)(IN_THREADS / 32) * DA_T * 4 * 32 * 8;
  const double2* Dm = (p.dense != nullptr && doff >= 0 && dense_ok) ? p.dense + doff : nullptr;
  const long long dmat = dense_matrix_elems(n);  // one stored matrix
  unsigned dch = 0;
  // ---- b = pre(rhs), beta0 = ||b||, V_0 = b / beta0 (krylov.py:61-80)
  if (Dm) {
    dense_apply(p, Dm, n, job, r0, VB, VY, s_nact, S, q, CS, dch);
    T.tick(3);
  } else {
    const int vm[3] = {VB, VY, VA};
    run_program(p, job, layer, w, r0, S.pph, p.pre_nph, vm, s_nact, S, q, CS, &tseq, T);
  }
  for (int l = q; l < ni; l += CS) instance_init(p, job, r0 + l, n, VY, dred);
  csync();
  rebuild_active(p, job, r0, ni, S.act, &s_nact);

  for (int j = 0; j < p.max_iter && s_nact > 0; ++j) {
    const int nact = s_nact;
    if (j + 1 > p.cap) {  // basis capacity exhausted: the host retries with a larger capacity
      for (int a = 0; a < nact; ++a) {
        const int l = S.act[a];
        if (l % CS == q && tid == 0) {
          p.state[job * p.R + r0 + l] = 2;
          p.iters[job * p.R + r0 + l] = -1;
          atomicMax(p.err, 5);
        }
      }
      csync();
      rebuild_active(p, job, r0, ni, S.act, &s_nact);
      break;
    }
    if (Dm) {  // w = pre(op(V_j)) as one dense product
      dense_apply(p, Dm + dmat, n, job, r0, j, j + 1, nact, S, q, CS, dch);
      T.tick(3);
    } else {
      const int vm1[3] = {j, VT, VA};
      run_program(p, job, layer, w, r0, S.oph, p.op_nph, vm1, nact, S, q, CS, &tseq, T);
      const int vm2[3] = {VT, j + 1, VA};
      run_program(p, job, layer, w, r0, S.pph, p.pre_nph, vm2, nact, S, q, CS, &tseq, T);
      T.tick(7);
    }
    // ---- MGS Arnoldi + Givens for the instances this CTA owns (krylov.py:89-127)
    for (int a = 0; a < nact; ++a) {
      const int l = S.act[a];
      if (l % CS != q) continue;
      instance_arnoldi(p, job, r0 + l, j, n, dred);
    }
    T.tick(6);
    csync();
    rebuild_active(p, job, r0, ni, S.act, &s_nact);
    T.tick(5);
    if (T.on) atomicAdd((unsigned long long*)&g_in_t[10], 1ULL);
  }

  // ---- x = V_k y, traces = down + up (nested.py:153), owner CTA per instance
  for (int l = q; l < ni; l += CS) instance_final(p, job, r0 + l, n, w, S.pan);
  T.tick(9);
  if (T.on) atomicAdd((unsigned long long*)&g_in_t[11], (unsigned long long)(clock64() - tk_entry));
}

// ---------------------------------------------------------------------------------------------
// Whole-GPU inner GMRES (cooperative launch, one CTA per SM) for every (job, group of <= 8 instances)
// unit of a stage whose layers carry dense inner operators.  Every step is spread over all CTAs:
// rhs_pol elementwise, each dense product as (unit, row-tile range) passes of dense_pass, the Arnoldi /
// Givens / x = V y of an instance on its owner CTA; grid-wide barriers separate the steps.  Same
// arithmetic, per instance, as the cluster kernel's dense path.
#define COOP_MAXU 256
__global__ void __launch_bounds__(IN_THREADS, 1) inner_coop_kernel(const InnerParams p, int nunits) {
  cg::grid_group grid = cg::this_grid();
  Ticker T;
  T.on = p.tprof && blockIdx.x == 0 && threadIdx.x == 0;
  T.start();
  auto gsync = [&]() {
    T.tick(7);
    grid.sync();
    T.tick(5);
  };
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t region = (size_t)p.coop_region;
  unsigned char* ring = smem;
  uint64_t* dbar = reinterpret_cast<uint64_t*>(smem + region);
  double* dred = reinterpret_cast<double*>(dbar + 2 * DA_NS);
  int* utile = reinterpret_cast<int*>(dred + 64);     // [nunits + 1] tile prefix of the active units
  int* unact = utile + COOP_MAXU + 1;                 // [nunits] active instances
  unsigned char* uact = reinterpret_cast<unsigned char*>(unact + COOP_MAXU);  // [nunits][8] active local ids
  unsigned char* sst = uact + COOP_MAXU * 8;          // [nunits][8] instance states (1 = frozen/absent)
  double2* yv = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(sst + COOP_MAXU * 8) + 127) & ~(uintptr_t)127);

  const int tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int ngroups = (p.R + 7) >> 3;
  const int nIc = p.Lc - 1;
  const int VB = p.cap + 1, VY = p.cap + 2;
  if (tid == 0) {
    for (int i = 0; i < DA_NS; ++i) {
      mbar_init(&dbar[i], 1);
      mbar_init(&dbar[DA_NS + i], IN_THREADS / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // per-job info staged once (the chained job -> layer -> width/offset loads stay off the step paths)
  __shared__ int s_job[COOP_MAXU], s_w[COOP_MAXU];
  __shared__ long long s_doff[COOP_MAXU];
  const int njob_ = nunits / ngroups;
  for (int jx = tid; jx < njob_; jx += blockDim.x) {
    const int job = p.stage_jobs[jx];
    const int layer = p.jobs[job].layer;
    s_job[jx] = job;
    s_w[jx] = p.layers[layer].w;
    s_doff[jx] = p.layers[layer].dense_off;
  }
  __syncthreads();
  // every instance's state, loaded by all threads in parallel
  auto load_states = [&](bool all) {
    for (int t = tid; t < nunits * 8; t += blockDim.x) {
      const int u = t >> 3, l = t & 7;
      const int r0_ = (u % ngroups) * 8;
      const bool ex = l < min(8, p.R - r0_);
      sst[t] = !ex ? 1 : (all ? 0 : (__ldcg(p.state + s_job[u / ngroups] * p.R + r0_ + l) == 0 ? 0 : 1));
    }
    __syncthreads();
  };
  auto ujob = [&](int u) { return s_job[u / ngroups]; };
  auto ur0 = [&](int u) { return (u % ngroups) * 8; };
  auto uni = [&](int u) { return min(8, p.R - (u % ngroups) * 8); };
  auto uw = [&](int u) { return s_w[u / ngroups]; };
  const int lane_ = tid & 31, wp_ = tid >> 5;
  (void)lane_;
  if (p.fused) {
    // ---- gather the job panels (k_gather_panels), then the pass-0 product (k_pass0): two 4-warp
    // items per CTA step, each with its own named barrier and partial-sum area in the ring region
    const long long tot = (long long)nunits / ngroups * 4 * p.R * p.wx;
    for (long long e = (long long)b * blockDim.x + tid; e < tot; e += (long long)G * blockDim.x)
      gather_elem(p.jobs, p.tab, p.rmap, p.R, p.wx, p.P, e);
    gsync();
    const int mp8 = q0_rows(p.wmax, p.kmax) / 8;
    const int gz0 = (p.maxj * p.R + P0_COLS - 1) / P0_COLS;
    const long long n0items = (long long)p.ngl * p.Lc * mp8 * gz0;
    const int half = wp_ >> 2;
    double* part = reinterpret_cast<double*>(ring) + half * (P0_KQ - 1) * 2 * 4 * 32;
    for (long long it = (long long)b * 2 + half; it < n0items + 1; it += (long long)G * 2) {
      if (it >= n0items) break;
      long long rest = it;
      const int z = (int)(rest % gz0);
      rest /= gz0;
      const int tile = (int)(rest % mp8);
      rest /= mp8;
      const int cc = (int)(rest % p.Lc), g = (int)(rest / p.Lc);
      pass0_item(p.grp, p.ljobs, p.jobs, p.cells, p.layers, p.q0, p.P, const_cast<double2*>(p.tables), p.smp, p.R, p.Lc,
                 p.wx, p.wmax, g,
                 cc, tile, z, wp_ & 3, part, 1 + half);
    }
    // generic-proxy writes to the ring must be ordered before the bulk copies of the dense products
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    gsync();
  }
  unsigned dch = 0;
  // y = M_which x over the active instances of every unit; all = every instance (the first product)
  // nmat > 1: `which` is a stack of nmat matrices sharing x (row tiles stacked), outputs dst, dst + 1, ...
  // Work list: (tile, active unit) pairs, TILE-major within a job (f = job base + tile * nA + unit index), so a
  // CTA streams the same operator tiles for every RHS group of a job back to back (the repeats hit L2).
  __shared__ short s_ug[COOP_MAXU][2];  // per unit: active units of its job, its index among them
  auto coop_apply = [&](int which, int src, int dst, bool all, int nmat = 1) {
    T.tick(7);
    load_states(all);
    if (tid == 0) {
      int tot = 0;
      for (int u = 0; u < nunits; ++u) {
        int na = 0;
        for (int l = 0; l < 8; ++l)
          if (sst[u * 8 + l] == 0) uact[u * 8 + na++] = (unsigned char)l;
        unact[u] = na;
      }
      for (int u0 = 0; u0 < nunits; u0 += ngroups) {  // one job: units u0 .. u0 + ngroups - 1
        int nA = 0;
        for (int g = 0; g < ngroups; ++g)
          if (unact[u0 + g] > 0) s_ug[u0 + g][1] = (short)nA++;
        // unit-major order for jobs of <= 2 RHS groups (PT_UNIT_MAJOR forces it): there the tile-major split halves
        // each pass and its staging overhead outweighs the L2 reuse (cfg2); from 3 groups on the reuse wins
        // (cfg3, 8 groups: 536 -> 497 ms per 64-source step)
        if (p.unit_major || ngroups <= 2) {  // each active unit its own contiguous range
          for (int g = 0; g < ngroups; ++g) {
            s_ug[u0 + g][0] = 1;
            s_ug[u0 + g][1] = 0;
            utile[u0 + g] = tot;
            if (unact[u0 + g] > 0) tot += nmat * ((4 * nIc * uw(u0) + 7) >> 3);
          }
          continue;
        }
        for (int g = 0; g < ngroups; ++g) {
          s_ug[u0 + g][0] = (short)nA;
          utile[u0 + g] = tot;
        }
        tot += nA * nmat * ((4 * nIc * uw(u0) + 7) >> 3);
      }
      utile[nunits] = tot;
    }
    __syncthreads();
    const int tot = utile[nunits];
    const int lo = (int)((long long)b * tot / G), hi = (int)((long long)(b + 1) * tot / G);
    auto cdivs = [](int a, int d) { return a <= 0 ? -((-a) / d) : (a + d - 1) / d; };
    for (int u = 0; u < nunits && lo < hi; ++u) {
      const int na = unact[u];
      if (na == 0) continue;
      const int nA = s_ug[u][0], gi = s_ug[u][1], T8u = nmat * ((4 * nIc * uw(u) + 7) >> 3);
      const int t0 = max(0, cdivs(lo - utile[u] - gi, nA)), t1 = min(T8u, cdivs(hi - utile[u] - gi, nA));
      if (t0 >= t1) continue;
      const int job = ujob(u), r0 = ur0(u), w = uw(u), n = 4 * nIc * w;
      int rr[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rr[i] = i < na ? r0 + uact[u * 8 + i] : r0;
      const double2* Mt = p.dense + s_doff[u / ngroups] + (size_t)which * dense_matrix_elems(n);
      T.tick(12);
      dense_pass(p, Mt, n, job, rr, na, src, dst, t0, t1, ring, region, dbar, dch, 8, nmat);
      T.tick(13);
    }
  };
  // ---- rhs_pol from the Newton tables (sie.py:230-242, negated), unless the pass-0 product wrote it already
  if (!p.rhs_ready || p.fused) {
    for (int u = 0; u < nunits; ++u) {
      const int job = ujob(u), r0 = ur0(u), ni = uni(u), w = uw(u), n = 4 * nIc * w;
      for (long long t = (long long)b * blockDim.x + tid; t < (long long)ni * n; t += (long long)G * blockDim.x) {
        const int l = (int)(t / n), e = (int)(t - (long long)l * n), r = r0 + l;
        const int seg = e / w, j = e - seg * w;
        const int half = seg / (2 * nIc);  // 0 down, 1 up
        const int I = (seg % (2 * nIc)) / 2, s_ = seg & 1;
        const int c = half == 0 ? I : I + 1;
        const int idx = half == 0 ? 2 + s_ : s_;
        const double2 tv = __ldcg(p.tables + ((((size_t)job * p.Lc + c) * 4 + idx) * p.R + r) * p.wmax + j);
        vecp(p, job, r, VB)[e] = make_double2(-tv.x, -tv.y);
      }
    }
    gsync();
  }
  // ---- b = pre(rhs) (krylov.py:61); s-step start: E b and E^2 b in the same pass, then Arnoldi steps 0-1
  T.tick(8);
  const int VT = p.cap + 3, VA = p.cap + 4;
  if (p.sstep)
    coop_apply(2, VB, VY, true, 3);  // [pre; E pre; E^2 pre] stacked: b, E b, E^2 b -> VY, VT, VA in one pass
  else
    coop_apply(0, VB, VY, true);
  T.tick(3);
  gsync();
  if (p.sstep) {
    for (int t = b; t < nunits * 8; t += G) {
      const int u = t >> 3, l = t & 7;
      if (l >= uni(u)) continue;
      const int n_ = 4 * nIc * uw(u);
      if (n_ <= 4 * IN_THREADS)
        instance_sstep(p, ujob(u), ur0(u) + l, n_, VY, VT, VA, dred, reinterpret_cast<double2*>(ring));
      else
        instance_sstep_loop(p, ujob(u), ur0(u) + l, n_, VY, VT, VA, dred);
    }
    T.tick(6);
    gsync();
  }
  for (int j = p.sstep ? 2 : 0; j < p.max_iter; ++j) {
    if (j > 0) {  // at j = 0 every instance enters (its state is set by the first Arnoldi step)
      load_states(false);
      int any = 0;
      for (int t = tid; t < nunits * 8; t += blockDim.x) any |= sst[t] == 0;
      if (!__syncthreads_or(any)) break;
    }
    if (j + 1 > p.cap) {  // basis capacity exhausted: the host retries with a larger capacity
      for (int t = b; t < nunits * 8; t += G) {
        const int u = t >> 3, l = t & 7;
        if (tid == 0 && l < uni(u)) {
          const int r = ur0(u) + l, job = ujob(u);
          if (__ldcg(p.state + job * p.R + r) == 0) {
            p.state[job * p.R + r] = 2;
            p.iters[job * p.R + r] = -1;
            atomicMax(p.err, 5);
          }
        }
      }
      gsync();
      break;
    }
    T.tick(4);  // loop head (active scan)
    // w = pre(op(V_j)); at j = 0 on the unnormalized b (every instance: beta0 is taken in the Arnoldi step)
    coop_apply(1, j == 0 ? VY : j, j + 1, j == 0);
    T.tick(3);
    gsync();
    for (int t = b; t < nunits * 8; t += G) {
      const int u = t >> 3, l = t & 7;
      if (l >= uni(u)) continue;
      const int job = ujob(u), r = ur0(u) + l;
      if (j == 0)
        instance_arnoldi0(p, job, r, 4 * nIc * uw(u), VY, dred);
      else if (__ldcg(p.state + job * p.R + r) == 0)
        instance_arnoldi(p, job, r, j, 4 * nIc * uw(u), dred);
    }
    T.tick(6);
    gsync();
  }
  for (int t = b; t < nunits * 8; t += G) {
    const int u = t >> 3, l = t & 7;
    // (instances the s-step already finalized, state 3, are skipped)
    if (l < uni(u) && p.state[ujob(u) * p.R + ur0(u) + l] != 3)
      instance_final(p, ujob(u), ur0(u) + l, 4 * nIc * uw(u), uw(u), yv);
  }
  T.tick(9);
  if (p.fused) {
    // ---- sampled trace response (k_green_samples) on the fresh traces, then the combination (k_combine)
    gsync();
    const int J = nunits / ngroups;
    const int gy = (p.R + 7) / 8;
    const int gzg = (p.kmax * 4 + 8 * GS_WARPS - 1) / (8 * GS_WARPS);
    const long long ngitems = (long long)J * p.Lc * gy * gzg;
    double2* trs = reinterpret_cast<double2*>(ring);
    for (long long it = b; it < ngitems; it += G) {
      const int z = (int)(it % gzg);
      const long long rest = it / gzg;
      const int y = (int)(rest % gy), x = (int)(rest / gy);
      green_item(p.jobs, p.cells, p.layers, p.gsmp, p.tr, p.smp, p.R, p.Lc, p.wx, p.wmax, x, y, z, trs);
    }
    gsync();
    const long long tot = (long long)J * 4 * p.R * p.wx;
    for (long long e = (long long)b * blockDim.x + tid; e < tot; e += (long long)G * blockDim.x)
      combine_elem(p.jobs, p.tab, p.rmap, p.R, p.wx, p.smp, e);
  }
}

// ---------------------------------------------------------------------------------------------
// Whole-GPU inner GMRES over the Green-block item programs (no dense operators; Lc > 8): the cluster
// kernel's arithmetic (item_unit, instance_init / instance_arnoldi / instance_final) with every CTA of the
// GPU sharing each program phase across all (job, <= 8 RHS) units of the stage, grid barriers between the
// phases.  A sweep stage's single unit then streams its Green tiles with the whole GPU's bandwidth instead
// of one 16-CTA cluster's.
#define CI_STATIC_INTS 0
__global__ void __launch_bounds__(IN_THREADS, 1) inner_coop_items_kernel(const InnerParams p, int nunits) {
  cg::grid_group grid = cg::this_grid();
  Ticker T;
  T.on = p.tprof && blockIdx.x == 0 && threadIdx.x == 0;
  T.start();
  auto gsync = [&]() {
    T.tick(7);
    grid.sync();
    T.tick(5);
  };
  extern __shared__ __align__(128) unsigned char smem[];
  InSmem S;
  S.tiles = reinterpret_cast<double2*>(smem);
  S.pan = S.tiles + (size_t)p.tring * p.wmax * 8;
  S.pan2 = S.pan + (size_t)4 * p.wmax * 8;
  S.red = S.pan2 + (size_t)2 * p.wmax * 8;
  double* dred = reinterpret_cast<double*>(S.red + (IN_THREADS / 32) * IN_MG * 8 * 8);
  S.tbar = reinterpret_cast<uint64_t*>(dred + 64);
  S.dbar = S.tbar + IN_TRMAX;
  int* uact = reinterpret_cast<int*>(S.dbar + 2 * DA_NS);  // [COOP_MAXU][8] active local ids per unit
  int* unact = uact + COOP_MAXU * 8;                       // [COOP_MAXU] active count per unit
  int* upre = unact + COOP_MAXU;                           // [COOP_MAXU + 1] prefix of active x ngrp
  int* oph = upre + COOP_MAXU + 1;
  int* pph = oph + 2 * PT_MAX_LC + 2;
  S.items = reinterpret_cast<IItem*>(pph + 2 * PT_MAX_LC + 2);
  S.act = nullptr;
  S.goff = nullptr;
  S.oph = oph;
  S.pph = pph;
  __shared__ int s_job[COOP_MAXU], s_w[COOP_MAXU], s_layer[COOP_MAXU];
  __shared__ short s_alist[COOP_MAXU];    // active units, job-major
  __shared__ int s_jstart[COOP_MAXU + 1];  // per job: start of its active units in s_alist
  const int tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const int ngroups = (p.R + 7) >> 3;
  const int nIc = p.Lc - 1;
  const int VB = p.cap + 1, VY = p.cap + 2, VT = p.cap + 3, VA = p.cap + 4;
  if (tid == 0) {
    for (int i = 0; i < IN_TRMAX; ++i) mbar_init(&S.tbar[i], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < p.nitems; i += blockDim.x) S.items[i] = p.items[i];
  for (int i = tid; i <= p.op_nph; i += blockDim.x) oph[i] = p.op_ph[i];
  for (int i = tid; i <= p.pre_nph; i += blockDim.x) pph[i] = p.pre_ph[i];
  const int njob_ = nunits / ngroups;
  for (int jx = tid; jx < njob_; jx += blockDim.x) {
    const int job = p.stage_jobs[jx];
    const int layer = p.jobs[job].layer;
    s_job[jx] = job;
    s_layer[jx] = layer;
    s_w[jx] = p.layers[layer].w;
  }
  __syncthreads();
  auto ujob = [&](int u) { return s_job[u / ngroups]; };
  auto ur0 = [&](int u) { return (u % ngroups) * 8; };
  auto uni = [&](int u) { return min(8, p.R - (u % ngroups) * 8); };
  auto uw = [&](int u) { return s_w[u / ngroups]; };
  auto ungrp = [&](int u) { return (((uw(u) + 7) >> 3) + p.mg - 1) / p.mg; };
  // active local instances of every unit, from the global states (all = every existing instance)
  auto refresh = [&](bool all) {
    for (int u = tid; u < nunits; u += blockDim.x) {
      int na = 0;
      const int r0 = ur0(u), ni = uni(u), job = ujob(u);
      for (int l = 0; l < ni; ++l)
        if (all || __ldcg(p.state + job * p.R + r0 + l) == 0) uact[u * 8 + na++] = l;
      unact[u] = na;
    }
    __syncthreads();
    if (tid == 0) {
      // per job: prefix (upre, indexed by job) of active units x tile groups, and its active units in order
      int acc = 0, na_tot = 0;
      for (int jx = 0; jx < njob_; ++jx) {
        upre[jx] = acc;
        s_jstart[jx] = na_tot;
        for (int g = 0; g < ngroups; ++g) {
          const int u = jx * ngroups + g;
          if (unact[u] > 0) {
            s_alist[na_tot++] = (short)u;
            acc += ungrp(u);
          }
        }
      }
      upre[njob_] = acc;
      s_jstart[njob_] = na_tot;
    }
    __syncthreads();
  };
  uint32_t tseq = 0;
  auto cdiv = [](long long a, long long bb) -> long long { return a <= 0 ? -((-a) / bb) : (a + bb - 1) / bb; };
  // one program over every unit's active instances: CTA b takes the (job, item, unit, tile group) work whose
  // weight midpoints fall in its share, job-major then item-major, so the RHS groups of a job run an item's
  // tile groups back to back on one CTA (their Green tiles repeat from L2); a grid barrier ends each phase
  // this CTA's work of phase phz in order, as cb(jx, ii, gi, u, g0, g1, item, goff) -> keep going?
  auto for_work = [&](const int* ph, int phz, auto&& cb) {
    const int it0 = ph[phz], nit = ph[phz + 1] - it0;
    int witems = 0;
    for (int ii = 0; ii < nit; ++ii) witems += S.items[it0 + ii].wgt;
    const long long wtot = (long long)upre[njob_] * witems;
    const long long wlo2 = 2 * ((long long)b * wtot / G), whi2 = 2 * ((long long)(b + 1) * wtot / G);
    // first job whose weight range reaches this CTA's share
    int lo = 0, hi = njob_;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (2LL * upre[mid + 1] * witems <= wlo2) lo = mid + 1;
      else hi = mid;
    }
    for (int jx = lo; jx < njob_ && 2LL * upre[jx] * witems < whi2; ++jx) {
      const int nA = s_jstart[jx + 1] - s_jstart[jx];
      if (nA == 0) continue;
      const int u_first = s_alist[s_jstart[jx]];
      const int ng = ungrp(u_first), layer = s_layer[jx];
      long long ib = (long long)upre[jx] * witems;  // item block start
      for (int ii = 0; ii < nit; ++ii) {
        const IItem& item = S.items[it0 + ii];
        const int wi = item.wgt;
        const long long iblock = (long long)wi * ng * nA;
        if (2 * (ib + iblock) <= wlo2 || 2 * ib >= whi2) {
          ib += iblock;
          continue;
        }
        const long long goff = p.cells[layer * p.Lc + (item.cell >= 0 ? item.cell : 0)].green_off;
        for (int gi = 0; gi < nA; ++gi) {
          const long long wa = ib + (long long)gi * wi * ng;
          const int g0 = (int)max(0LL, cdiv(wlo2 - 2 * wa - wi, 2LL * wi));
          const int g1 = (int)min((long long)ng, cdiv(whi2 - 2 * wa - wi, 2LL * wi));
          if (g0 >= g1) continue;
          if (!cb(jx, ii, gi, s_alist[s_jstart[jx] + gi], g0, g1, item, goff)) return;
        }
        ib += iblock;
      }
    }
  };
  // one program over every unit's active instances: CTA b takes the (job, item, unit, tile group) work whose
  // weight midpoints fall in its share, job-major then item-major, so the RHS groups of a job run an item's
  // tile groups back to back on one CTA (their Green tiles repeat from L2); a grid barrier ends each phase.
  // With p.tprefetch (opt-in) a CTA issues, before the barrier, the first Green tiles of its first work item of
  // the next phase (operator data, independent of the phase results).
  auto coop_program = [&](const int* ph, int nph, const int vmap[3]) {
    int pf_phz = -1, pf_jx = -1, pf_ii = -1, pf_gi = -1, pf_n = 0;
    for (int phz = 0; phz < nph; ++phz) {
      bool first = true;
      for_work(ph, phz, [&](int jx, int ii, int gi, int u, int g0, int g1, const IItem& item, long long goff) {
        const int pre = (first && pf_phz == phz && jx == pf_jx && ii == pf_ii && gi == pf_gi) ? pf_n : 0;
        first = false;
        T.tick(12);
        item_unit(p, ujob(u), uw(u), ur0(u), uact + u * 8, unact[u], item, g0, g1, vmap, S, &tseq, T, goff, pre);
        return true;
      });
      pf_phz = -1;
      pf_n = 0;
      if (p.tprefetch && phz + 1 < nph)
        for_work(ph, phz + 1, [&](int jx, int ii, int gi, int u, int g0, int g1, const IItem& item, long long goff) {
          if (tid == 0) pf_n = item_prefetch(p, uw(u), item, g0, g1, S, &tseq, goff);
          pf_phz = phz + 1;
          pf_jx = jx;
          pf_ii = ii;
          pf_gi = gi;
          return false;  // the first work item only
        });
      gsync();
    }
  };
  // ---- rhs_pol from the Newton tables (sie.py:230-242, negated)
  for (int u = 0; u < nunits; ++u) {
    const int job = ujob(u), r0 = ur0(u), ni = uni(u), w = uw(u), n = 4 * nIc * w;
    for (long long t = (long long)b * blockDim.x + tid; t < (long long)ni * n; t += (long long)G * blockDim.x) {
      const int l = (int)(t / n), e = (int)(t - (long long)l * n), r = r0 + l;
      const int seg = e / w, j = e - seg * w;
      const int half = seg / (2 * nIc);
      const int I = (seg % (2 * nIc)) / 2, s_ = seg & 1;
      const int c = half == 0 ? I : I + 1;
      const int idx = half == 0 ? 2 + s_ : s_;
      const double2 tv = __ldcg(p.tables + ((((size_t)job * p.Lc + c) * 4 + idx) * p.R + r) * p.wmax + j);
      vecp(p, job, r, VB)[e] = make_double2(-tv.x, -tv.y);
    }
  }
  refresh(true);
  gsync();
  T.tick(8);
  // ---- b = pre(rhs), beta0 = ||b||, V_0 = b / beta0 (krylov.py:61-80)
  {
    const int vm[3] = {VB, VY, VA};
    coop_program(pph, p.pre_nph, vm);
  }
  for (int t = b; t < nunits * 8; t += G) {
    const int u = t >> 3, l = t & 7;
    if (l < uni(u)) instance_init(p, ujob(u), ur0(u) + l, 4 * nIc * uw(u), VY, dred);
  }
  gsync();
  for (int j = 0; j < p.max_iter; ++j) {
    refresh(false);
    if (upre[njob_] == 0) break;
    if (j + 1 > p.cap) {  // basis capacity exhausted: the host retries with a larger capacity
      for (int t = b; t < nunits * 8; t += G) {
        const int u = t >> 3, l = t & 7;
        if (tid == 0 && l < uni(u)) {
          const int r = ur0(u) + l, job = ujob(u);
          if (__ldcg(p.state + job * p.R + r) == 0) {
            p.state[job * p.R + r] = 2;
            p.iters[job * p.R + r] = -1;
            atomicMax(p.err, 5);
          }
        }
      }
      gsync();
      break;
    }
    T.tick(4);
    {
      const int vm1[3] = {j, VT, VA};
      coop_program(oph, p.op_nph, vm1);
      const int vm2[3] = {VT, j + 1, VA};
      coop_program(pph, p.pre_nph, vm2);
    }
    T.tick(3);
    for (int t = b; t < nunits * 8; t += G) {
      const int u = t >> 3, l = t & 7;
      if (l >= uni(u)) continue;
      const int job = ujob(u), r = ur0(u) + l;
      if (__ldcg(p.state + job * p.R + r) == 0) instance_arnoldi(p, job, r, j, 4 * nIc * uw(u), dred);
    }
    T.tick(6);
    gsync();
  }
  for (int t = b; t < nunits * 8; t += G) {
    const int u = t >> 3, l = t & 7;
    if (l < uni(u)) instance_final(p, ujob(u), ur0(u) + l, 4 * nIc * uw(u), uw(u), S.pan);
  }
  T.tick(9);
}

int inner_coop_max_units() { return COOP_MAXU; }

size_t inner_coop_smem(const InnerParams& p, size_t region) {
  return region + 2 * DA_NS * 8 + 64 * 8 + (COOP_MAXU + 1) * 4 + COOP_MAXU * 4 + 2 * COOP_MAXU * 8 + 128 +
         (size_t)(p.cap + 2 + 24 + 300 + 24) * 16 + 128;
}

// extra shared memory of the cooperative item kernel over the cluster kernel's layout
static size_t coop_items_extra() { return (size_t)COOP_MAXU * 8 * 4 + COOP_MAXU * 4 + (COOP_MAXU + 1) * 4; }

static cudaError_t inner_coop_items_launch(const InnerParams& p0, int njobs, cudaStream_t st) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int nunits = njobs * ((p0.R + 7) / 8);
  if (nunits > COOP_MAXU || p0.Lc < 2 || std::getenv("PT_NO_COOP_ITEMS")) return cudaErrorNotSupported;
  InnerParams p = p0;
  // the ring gives up what the unit tables take (static s_job/s_w/s_layer: 3 COOP_MAXU ints)
  const int w = p.wmax < 8 ? 8 : p.wmax;
  const long long tb = (long long)w * 8 * 16;
  const long long shrink = ((long long)coop_items_extra() + 5LL * COOP_MAXU * 4 + tb - 1) / tb;
  p.tring = (int)std::min((long long)IN_TRMAX, (long long)inner_tring(p.wmax, p.nitems) - shrink);
  if (p.tring < 4 * p.mg) p.mg = 1;
  if (p.tring < 4) return cudaErrorNotSupported;
  const size_t sm = inner_smem_bytes(p.wmax, p.nitems, p.tring) + coop_items_extra();
  set_smem_attr((const void*)inner_coop_items_kernel, sm);
  static std::unordered_map<size_t, int> occ;
  auto it = occ.find(sm);
  if (it == occ.end()) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inner_coop_items_kernel, IN_THREADS, sm);
    cudaGetLastError();
    it = occ.emplace(sm, per_sm).first;
  }
  if (it->second < 1) return cudaErrorNotSupported;
  int nu = nunits;
  void* args[] = {(void*)&p, (void*)&nu};
  const int grid = p.coop_sms > 0 ? std::min(nsm, p.coop_sms) : nsm;
  return cudaLaunchCooperativeKernel((const void*)inner_coop_items_kernel, dim3(grid), dim3(IN_THREADS), args, sm, st);
}

// returns cudaErrorNotSupported when the cooperative path does not apply (caller falls back)
cudaError_t inner_coop_launch(const InnerParams& p0, int njobs, cudaStream_t st) {
  if (!p0.dense) {
    const cudaError_t e = inner_items_launch(p0, njobs, st);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
    return inner_coop_items_launch(p0, njobs, st);
  }
  static int nsm = 0, maxsm = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!nsm) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  const int nunits = njobs * ((p0.R + 7) / 8);
  if (!p0.dense || nunits > COOP_MAXU || p0.Lc < 2) return cudaErrorNotSupported;
  InnerParams p = p0;
  // ring: as many DA_KC-chunk slots as fit next to the small arrays and the kernel's static shared memory
  // (>= 2), and >= the partial tiles
  static size_t static_sm = (size_t)-1;
  if (static_sm == (size_t)-1) {
    cudaFuncAttributes fa;
    static_sm = cudaFuncGetAttributes(&fa, inner_coop_kernel) == cudaSuccess ? fa.sharedSizeBytes : 16384;
  }
  size_t slot = (size_t)DA_T * DA_KC * 512 + 8 * (8 * DA_KC * 4 + 4) * 16;  // dense_slot_bytes(8)
  const size_t fixed = inner_coop_smem(p, 0) + static_sm;
  // PT_DA_NS = n: n equal slots filling the shared memory left (each >= one 8-tile chunk + 8 x rows)
  static const int da_ns = std::getenv("PT_DA_NS") ? atoi(std::getenv("PT_DA_NS")) : 0;
  if (da_ns >= 2 && da_ns <= DA_NS) {
    const size_t s2 = ((size_t)maxsm - fixed) / da_ns / 128 * 128;
    if (s2 >= (size_t)DA_T * DA_KC * 512 + 8 * (DA_KC * 4 + 4) * 16) slot = s2;
  }
  p.da_slot = (int)slot;
  size_t region = std::min((size_t)DA_NS * slot, ((size_t)maxsm - fixed) / slot * slot);
  if (region < 2 * slot || region < (size_t)(IN_THREADS / 32) * DA_T * 4 * 32 * 8) return cudaErrorNotSupported;
  if (p.fused && (region < (size_t)4 * ((p.wmax + 3) & ~3) * 8 * 16 || region < 2 * (P0_KQ - 1) * 2 * 4 * 32 * 8))
    return cudaErrorNotSupported;
  p.coop_region = (long long)region;
  const size_t sm = inner_coop_smem(p, region);
  set_smem_attr((const void*)inner_coop_kernel, sm);
  static std::unordered_map<size_t, int> occ;  // co-residency per shared-memory size (queried once)
  auto it = occ.find(sm);
  if (it == occ.end()) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inner_coop_kernel, IN_THREADS, sm);
    it = occ.emplace(sm, per_sm).first;
  }
  if (it->second < 1) return cudaErrorNotSupported;
  const int grid = p.coop_sms > 0 ? std::min(nsm, p.coop_sms) : nsm;  // one CTA per SM (of the budget)
  void* args[] = {(void*)&p, (void*)&nunits};
  int nu = nunits;
  args[1] = (void*)&nu;
  return cudaLaunchCooperativeKernel((const void*)inner_coop_kernel, dim3(grid), dim3(IN_THREADS), args, sm, st);
}

int inner_mg(int wmax) { return wmax <= 80 ? 2 : 1; }

// shared memory of the cluster kernel without its Green-tile ring
static size_t inner_smem_fixed(int wmax, int nitems) {
  const int w = wmax < 8 ? 8 : wmax;
  return (size_t)(4 + 2) * w * 8 * 16 + (size_t)(IN_THREADS / 32) * IN_MG * 8 * 8 * 16 + 64 * 8 + IN_TRMAX * 8 +
         2 * DA_NS * 8 + 64 + PT_MAX_LC * 8 + 2 * (2 * PT_MAX_LC + 2) * 4 + (size_t)nitems * sizeof(IItem) + 128;
}

// Green-tile ring slots: as many single tiles (8 rows x w) as fit next to the rest (<= IN_TRMAX, >= 2)
int inner_tring(int wmax, int nitems) {
  static int maxsm = 0;
  if (!maxsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  const int w = wmax < 8 ? 8 : wmax;
  // (static __shared__ of the kernel and alignment slack come off the opt-in limit)
  long long room = (long long)maxsm - 8192 - (long long)inner_smem_fixed(wmax, nitems);
  if (const char* e = std::getenv("PT_TRING")) room = std::min(room, (long long)atoi(e) * w * 8 * 16);
  const long long t = room / ((long long)w * 8 * 16);
  return (int)std::max(0LL, std::min((long long)IN_TRMAX, t));
}

size_t inner_smem_bytes(int wmax, int nitems, int tring) {
  const int w = wmax < 8 ? 8 : wmax;
  return inner_smem_fixed(wmax, nitems) + (size_t)tring * w * 8 * 16;
}

cudaError_t inner_launch(const InnerParams& p, int njobs, cudaStream_t st) {
  if (njobs == 0 || p.Lc < 2) return cudaSuccess;
  if (p.tring < 4 * p.mg) {  // program items do not fit in shared memory
    fprintf(stderr, "inner_launch: %d program items leave no room for the Green-tile ring\n", p.nitems);
    return cudaErrorInvalidValue;
  }
  const size_t sm = inner_smem_bytes(p.wmax, p.nitems, p.tring);
  set_smem_attr((const void*)inner_gmres_kernel, sm);
  static bool nonportable = false;
  if (!nonportable) {
    cudaFuncSetAttribute(inner_gmres_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    nonportable = true;
  }
  const int ngroups = (p.R + 7) / 8;
  const int nclusters = njobs * ngroups;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(IN_THREADS, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // Clusters of 16 CTAs (twice the FP64 tensor throughput per RHS group) when they all fit at once;
  // otherwise the portable 8.  PT_INNER_CS overrides.
  int cs = INNER_CS;
  static int occ1 = -1;  // co-resident CTAs per SM at this kernel's shared-memory size
  if (occ1 < 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, inner_gmres_kernel, IN_THREADS, sm);
    cudaGetLastError();
    occ1 = std::max(occ1, 1);
  }
  if (const char* e = std::getenv("PT_INNER_CS")) {
    const int v = atoi(e);
    cs = v >= 16 ? 16 : (v >= 8 ? 8 : (v >= 4 ? 4 : (v >= 2 ? 2 : 1)));
  } else if (nclusters * 16 <= nsm * occ1) {
    // (smaller clusters over more waves were measured slower: a unit's phases are latency-bound, cfg4
    // 9.3 / 16.2 / 25.6 s per 256-source step at 8 / 4 / 2 CTAs per cluster)
    cfg.gridDim = dim3(nclusters * 16, 1, 1);
    attr[0].val.clusterDim.x = 16;
    static std::unordered_map<size_t, int> act16;  // co-resident 16-CTA clusters per shared-memory size
    auto it = act16.find(sm);
    if (it == act16.end()) {
      int active = 0;
      if (cudaOccupancyMaxActiveClusters(&active, inner_gmres_kernel, &cfg) != cudaSuccess) active = 0;
      cudaGetLastError();
      it = act16.emplace(sm, active).first;
    }
    if (it->second >= nclusters) cs = 16;
  }
  cfg.gridDim = dim3(nclusters * cs, 1, 1);
  attr[0].val.clusterDim.x = cs;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, inner_gmres_kernel, p);
  if (e != cudaSuccess)
    fprintf(stderr, "inner_launch: %s (smem %zu, tring %d, nitems %d, wmax %d, clusters %d x %d)\n",
            cudaGetErrorString(e), sm, p.tring, p.nitems, p.wmax, nclusters, cs);
  return e;
}

void inner_items_tprof_dump(const char* tag);
void inner_tprof_dump(const char* tag) {
  inner_items_tprof_dump(tag);
  long long t[16];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(t, g_in_t, sizeof(t));
  fprintf(stderr, "inner tprof [%s] (cycles, CTA 0): setup %lld tiles+prefetch %lld gather %lld tilewait %lld dmma %lld "
          "combine %lld cluster-bar %lld arnoldi %lld rest %lld final %lld | iterations %lld total %lld | bookkeeping %lld "
          "tile-issue %lld | dense data-wait (warp 1) %lld\n", tag, t[8], t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[9], t[10],
          t[11], t[12], t[13], t[14]);
  long long z[16] = {0};
  cudaMemcpyToSymbol(g_in_t, z, sizeof(z));
}
