// Host orchestration of the online stage and the C ABI (include/pt_b200.h).
//
// The outer left-preconditioned GMRES (krylov.py:53-135) is driven from here
// with ONE host synchronisation per outer iteration (the Hessenberg column);
// every layer-solve, inner Krylov iteration, Arnoldi reduction and the
// reconstruction run on the device.  The outer operator and preconditioner of
// sie.py:203-326 are encoded once, at pt_create, as "stages" of independent
// layer-solve jobs (OJob) plus small vector combinations; a stage executes as
//   gather panels -> K1 (Newton pass) -> inner GMRES -> K1 (reconstruction pass) -> combine.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/pt_b200.h"
#include "pt_launch.cuh"
#include "stage_dev.cuh"  // P0_KQ (k_inner_lu launch shape)

using cplx = std::complex<double>;

static thread_local std::string g_err;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      g_err = std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + std::to_string(__LINE__); \
      return PT_CUDA_ERROR;                                                                \
    }                                                                                      \
  } while (0)

namespace {

const Ref NOREF{-1, 0};

struct Stage {
  const char* name = "";  // for the PT_STAGE_PROF breakdown
  std::vector<OJob> jobs;
  OJob* jobs_d = nullptr;
  int* stage_jobs_d = nullptr;
  std::vector<int> ljobs;                 // job ids grouped by layer
  std::vector<std::pair<int, int>> lgrp;  // (layer, begin in ljobs); count from next
  int* ljobs_d = nullptr;
  bool any_panel = false, any_sample = false;
  bool samples_only = true;  // every job's outputs are layer-row samples (no volume output)
  bool no_volume = true;     // no job has a volume source
  int* grp_d = nullptr;      // [ngroups][3]: layer, first index into ljobs, job count
  // task cache per active-RHS count
  struct Tasks {
    K1Task* d = nullptr;
    int n = 0, nc = 1;
    long long zsize = 0;
    int cm = 1;
    double bytes = 0.0;  // algorithmic S^-1 bytes of one pass: 32 wz_c w^2 per (cell, column)
    double hbytes = 0.0; // S^-1 bytes one pass streams: 16 wz_c w^2 per task (a task serves its nq columns)
  };
  // executed work of one launch per active RHS (flops) and the operator bytes it streams, per kernel class
  bool work_ok = false;
  double p0_fpr = 0, p0_bytes = 0, gs_fpr = 0, gs_bytes = 0, in_bytes = 0;
  std::map<int, Tasks> tasks;
};

template <class T>
int upload(T** dst, const T* src, size_t n) {
  if (n == 0) {
    *dst = nullptr;
    return 0;
  }
  CK(cudaMalloc(dst, n * sizeof(T)));
  CK(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyDefault));
  return 0;
}

}  // namespace

#define PT_RMAP_SLOTS 32
struct pt_ctx {
  int dev = 0;
  cudaStream_t st = nullptr;
  int nx, nz, npml, L, Lc, wx, wz, nI, wmax, wzcmax;
  double h, omega;
  std::vector<LayerInfo> lay;
  std::vector<CellInfo> cel;
  LayerInfo* lay_d = nullptr;
  CellInfo* cel_d = nullptr;
  double2 *sinv_d = nullptr, *green_d = nullptr, *lz_d = nullptr, *uz_d = nullptr;
  double2* gsmp_d = nullptr;  // sampled trace responses (optional; enables the one-pass layer solve)
  double2* q0_d = nullptr;    // pass-0 operators (optional; layer solves without volume sources skip K1)
  double2* dense_d = nullptr; // dense inner operators (optional)
  double2* lu_d = nullptr;    // direct inner backend: per-layer A^-1 (optional, backend="lu")
  int dense_cnt = 2;          // dense matrices per layer (4: with the s-step operators)
  double2* tables_f = nullptr;  // Newton tables of the volume sources alone (NEWTON stage), reused by RECON
  bool tables_f_ok = false;
  int tables_f_R = 0;
  double2 *tx_d = nullptr, *tz_d = nullptr;
  double* m_d = nullptr;
  double2* hd_d = nullptr;  // optional global-operator diagonal for the residual
  // inner item programs
  IItem* items_d = nullptr;
  int *op_ph_d = nullptr, *pre_ph_d = nullptr;
  int op_nph = 0, pre_nph = 0, nitems = 0;
  long long op_blocks = 0, pre_blocks = 0;
  // scan form of the inner GS sweeps (single-job stages; see build_inner): product blocks in the Green pool and a
  // second preconditioner program
  int scan_levels = 0;  // product levels stored per cell (strides 2, 4, ...); 0 = none
  IItem* items_px_d = nullptr;
  int* pre_ph_px_d = nullptr;
  int pre_nph_px = 0, nitems_px = 0;
  // outer stages
  Stage newton, op, refl, recon, layer_solve;
  std::vector<Stage> sdown, sup;  // sdown[I] for I=1..nI-1, sup[I] for I=0..nI-2
  // solve scratch
  int capR = 0, capO = 0, inner_cap = 12;  // inner Krylov basis; grown (up to inner_max_iter + 1) on demand
  long long nO = 0;
  double2 *V = nullptr, *Bv = nullptr, *Bp = nullptr, *T1 = nullptr, *AX = nullptr, *X = nullptr, *TR = nullptr;
  double2 *P = nullptr, *smp = nullptr, *tables = nullptr, *trc = nullptr, *Z = nullptr, *iscr = nullptr,
          *hess = nullptr;
  long long zcap = 0, iscr_stride = 0, hstride = 0, inmax = 0;
  int* iters = nullptr;
  int* istate = nullptr;
  double* ibeta0 = nullptr;
  int* err_d = nullptr;
  unsigned long long* cnt_d = nullptr;  // [0] inner iterations, [1] touches, [2] instances
  int* hist_d = nullptr;
  int* rmap_d = nullptr;
  double *dscal = nullptr, *hnorm = nullptr;
  double2 *hout = nullptr, *ybuf = nullptr;
  int* hrmap = nullptr;
  double2 *io_f = nullptr, *io_u = nullptr;  // pt_solve staging buffers (reused)
  size_t io_bytes = 0;
  double2* hhout = nullptr;
  double* hdscal = nullptr;
  double2* hy = nullptr;
  // host view of current active set
  std::vector<int> act;
  int slot_bytes = 32768, ns = 8, num_sms = 148;
  long long layer_solves = 0;
  // stream + profiling
  cudaStream_t own_st = nullptr;
  bool prof = false;
  struct EvRec {
    cudaEvent_t a, b;
    int cls;  // 0 K1, 1 inner, 2 other, 3 sampled trace response, 4 pass-0 product (3, 4 counted as other)
    const char* tag;
  };
  const char* cur_tag = "";
  std::vector<cudaEvent_t> evpool;
  size_t ev_next = 0;
  std::vector<EvRec> evs;
  double k1_bytes = 0.0;
  long long launches = 0, k1_launches = 0;
  // CUDA graphs of the fixed launch sequences of a solve (graphed()): one executable per key, captured
  // the second time the key is seen (the first, eager run makes every lazy allocation); gen changes
  // whenever a buffer the sequences use is reallocated, which retires the old keys
  struct GraphEnt {
    int seen = 0;
    cudaGraphExec_t exec = nullptr;
    long long d_layer_solves = 0, d_launches = 0, d_k1_launches = 0, d_touch = 0;
    double d_k1_bytes = 0.0;
    double d_cf[5] = {0, 0, 0, 0, 0}, d_cb[5] = {0, 0, 0, 0, 0};
  };
  std::map<std::vector<long long>, GraphEnt> graphs;
  long long graphs_gen = -1;
  double cls_flops[5] = {0, 0, 0, 0, 0}, cls_bytes[5] = {0, 0, 0, 0, 0};  // executed work per kernel class
  double2* ipart = nullptr;  // vector-phase partials of the whole-GPU item-program inner kernel
  long long ipart_items = 0;  // buffer generation the cached executables were captured against
  long long gen = 0;
  bool graphs_off = false;
  int coop_sms = 0;  // SM budget of the cooperative inner kernels (PT_COOP_SMS; 0 = all)
  // outputs copied to the host while the reconstruction runs: side stream, events, pinned staging
  cudaStream_t side_st = nullptr;
  cudaEvent_t ev_tr = nullptr, ev_cp = nullptr;
  int batch_cap = 0;       // RHS per lockstep batch on the item-program path (decided at the first solve)
  int* zflag_d = nullptr;  // [L][R] nonzero-source flags of the NEWTON stage (k_slab_flags)
  int zflag_cap = 0;
  // pt_solve on host buffers, several lockstep batches: the copies of batch b +- 1 run on io_st while batch b solves
  cudaStream_t io_st = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_done = nullptr;
  double2* hstage = nullptr;
  size_t hstage_cap = 0;
  std::vector<long long> asm_touch;  // per layer: assembled-boundary touches per boundary_samples call
  long long touch_extra = 0;         // host-side touches of this solve (assembled boundary accounting)
  unsigned rmap_slot = 0;
};

static cudaEvent_t pool_event(pt_ctx* c) {
  if (c->ev_next == c->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->evpool.push_back(e);
  }
  return c->evpool[c->ev_next++];
}

// Counts every launch; with profiling on, brackets it with CUDA events on the launch stream.
struct LaunchScope {
  pt_ctx* c;
  int cls;
  cudaEvent_t a = nullptr;
  LaunchScope(pt_ctx* c_, int cls_) : c(c_), cls(cls_) {
    c->launches++;
    if (cls == 0) c->k1_launches++;
    if (c->prof) {
      a = pool_event(c);
      cudaEventRecord(a, c->st);
    }
  }
  ~LaunchScope() {
    if (c->prof) {
      cudaEvent_t b = pool_event(c);
      cudaEventRecord(b, c->st);
      c->evs.push_back({a, b, cls, c->cur_tag});
    }
  }
};

// ------------------------------------------------------------------ program builders

static int segD(const pt_ctx* c, int I, int s) { return 2 * I + s; }
static int segU(const pt_ctx* c, int I, int s) { return 2 * c->nI + 2 * I + s; }

static OJob blank_job(int layer) {
  OJob j;
  std::memset(&j, 0, sizeof(j));
  j.layer = layer;
  for (int s = 0; s < 4; ++s) {
    j.pan[s][0] = j.pan[s][1] = NOREF;
    j.dst[s] = j.add[s] = NOREF;
    j.sub[s][0] = j.sub[s][1] = NOREF;
    j.scoef[s] = 1.0;
  }
  return j;
}
static void add_out(OJob& j, int row, Ref dst, double scoef, Ref s0 = NOREF, Ref s1 = NOREF) {
  const int o = j.nout++;
  j.orow[o] = row;
  j.dst[o] = dst;
  j.scoef[o] = scoef;
  j.sub[o][0] = s0;
  j.sub[o][1] = s1;
}

static int finalize_stage(pt_ctx* c, Stage& S) {
  const int J = (int)S.jobs.size();
  std::vector<int> sj(J);
  for (int i = 0; i < J; ++i) sj[i] = i;
  S.ljobs.clear();
  S.lgrp.clear();
  for (int l = 0; l < c->L; ++l) {
    const int b = (int)S.ljobs.size();
    for (int i = 0; i < J; ++i)
      if (S.jobs[i].layer == l) S.ljobs.push_back(i);
    if ((int)S.ljobs.size() > b) S.lgrp.push_back({l, b});
  }
  for (auto& jb : S.jobs) {
    for (int s = 0; s < 4; ++s)
      if (jb.pan[s][0].vec >= 0) S.any_panel = true;
    if (jb.nout > 0) S.any_sample = true;
    if (jb.nout <= 0) S.samples_only = false;
    if (jb.vol) S.no_volume = false;
  }
  {
    std::vector<int> g;
    for (size_t i = 0; i < S.lgrp.size(); ++i) {
      const int b = S.lgrp[i].second;
      const int e = i + 1 < S.lgrp.size() ? S.lgrp[i + 1].second : (int)S.ljobs.size();
      g.push_back(S.lgrp[i].first);
      g.push_back(b);
      g.push_back(e - b);
    }
    if (!g.empty() && upload(&S.grp_d, g.data(), g.size())) return PT_CUDA_ERROR;
  }
  if (upload(&S.jobs_d, S.jobs.data(), S.jobs.size())) return PT_CUDA_ERROR;
  if (upload(&S.stage_jobs_d, sj.data(), sj.size())) return PT_CUDA_ERROR;
  if (upload(&S.ljobs_d, S.ljobs.data(), S.ljobs.size())) return PT_CUDA_ERROR;
  return 0;
}

// vec ids of outer stages: 0 IN, 1 OUT, 2 AUX
static int build_outer(pt_ctx* c) {
  const int L = c->L, nI = c->nI;
  // NEWTON (sie.py:175-188 + 230-242): rhs.down = -N_{n,n+1}, rhs.up = -N_{0,1}
  for (int l = 0; l < L; ++l) {
    OJob j = blank_job(l);
    j.vol = 1;
    const int n = c->lay[l].n;
    if (l >= 1) {
      add_out(j, 0, Ref{1, segU(c, l - 1, 0)}, -1.0);
      add_out(j, 1, Ref{1, segU(c, l - 1, 1)}, -1.0);
    }
    if (l <= L - 2) {
      add_out(j, n, Ref{1, segD(c, l, 0)}, -1.0);
      add_out(j, n + 1, Ref{1, segD(c, l, 1)}, -1.0);
    }
    if (j.nout > 0) c->newton.jobs.push_back(j);
  }
  // OP = apply_M_polarized (sie.py:203-228)
  for (int l = 0; l < L; ++l) {
    const bool top = l >= 1, bot = l <= L - 2;
    const int ib = l, it = l - 1;
    const int n = c->lay[l].n;
    if (bot) {
      OJob j = blank_job(l);
      if (top) {
        j.pan[0][0] = Ref{0, segD(c, ib - 1, 0)};
        j.pan[0][1] = Ref{0, segU(c, ib - 1, 0)};
        j.pan[1][0] = Ref{0, segD(c, ib - 1, 1)};
        j.pan[1][1] = Ref{0, segU(c, ib - 1, 1)};
      }
      j.pan[2][0] = Ref{0, segU(c, ib, 0)};
      j.pan[3][0] = Ref{0, segU(c, ib, 1)};
      add_out(j, n, Ref{1, segD(c, ib, 0)}, 1.0, Ref{0, segD(c, ib, 0)}, Ref{0, segU(c, ib, 0)});
      add_out(j, n + 1, Ref{1, segD(c, ib, 1)}, 1.0, Ref{0, segD(c, ib, 1)});
      c->op.jobs.push_back(j);
    }
    if (top) {
      OJob j = blank_job(l);
      j.pan[0][0] = Ref{0, segD(c, it, 0)};
      j.pan[1][0] = Ref{0, segD(c, it, 1)};
      if (bot) {
        j.pan[2][0] = Ref{0, segU(c, ib, 0)};
        j.pan[2][1] = Ref{0, segD(c, ib, 0)};
        j.pan[3][0] = Ref{0, segU(c, ib, 1)};
        j.pan[3][1] = Ref{0, segD(c, ib, 1)};
      }
      add_out(j, 0, Ref{1, segU(c, it, 0)}, 1.0, Ref{0, segU(c, it, 0)});
      add_out(j, 1, Ref{1, segU(c, it, 1)}, 1.0, Ref{0, segD(c, it, 1)}, Ref{0, segU(c, it, 1)});
      c->op.jobs.push_back(j);
    }
  }
  // sweep_down steps (sie.py:272-283): IN = v, OUT = y
  c->newton.name = "newton";
  c->op.name = "op";
  c->refl.name = "refl";
  c->recon.name = "recon";
  c->sdown.resize(std::max(nI, 1));
  for (auto& st : c->sdown) st.name = "sdown";
  for (int I = 1; I < nI; ++I) {
    OJob j = blank_job(I);
    const int n = c->lay[I].n;
    j.pan[0][0] = Ref{1, segD(c, I - 1, 0)};
    j.pan[1][0] = Ref{1, segD(c, I - 1, 1)};
    add_out(j, n, Ref{1, segD(c, I, 0)}, 1.0, Ref{0, segD(c, I, 0)});
    add_out(j, n + 1, Ref{1, segD(c, I, 1)}, 1.0, Ref{0, segD(c, I, 1)});
    c->sdown[I].jobs.push_back(j);
  }
  // upward_reflections (sie.py:298-308): IN = y (down half), OUT = aux (up half)
  for (int I = 0; I < nI; ++I) {
    OJob j = blank_job(I + 1);
    j.pan[0][0] = Ref{0, segD(c, I, 0)};
    j.pan[1][0] = Ref{0, segD(c, I, 1)};
    if (I <= nI - 2) {
      j.pan[2][0] = Ref{0, segD(c, I + 1, 0)};
      j.pan[3][0] = Ref{0, segD(c, I + 1, 1)};
    }
    add_out(j, 0, Ref{1, segU(c, I, 0)}, 1.0);
    add_out(j, 1, Ref{1, segU(c, I, 1)}, 1.0, Ref{0, segD(c, I, 1)});
    c->refl.jobs.push_back(j);
  }
  // sweep_up steps (sie.py:285-296): IN holds s in its up half, OUT = y
  c->sup.resize(std::max(nI, 1));
  for (auto& st : c->sup) st.name = "sup";
  for (int I = nI - 2; I >= 0; --I) {
    OJob j = blank_job(I + 1);
    j.pan[2][0] = Ref{1, segU(c, I + 1, 0)};
    j.pan[3][0] = Ref{1, segU(c, I + 1, 1)};
    add_out(j, 0, Ref{1, segU(c, I, 0)}, 1.0, Ref{0, segU(c, I, 0)});
    add_out(j, 1, Ref{1, segU(c, I, 1)}, 1.0, Ref{0, segU(c, I, 1)});
    c->sup[I].jobs.push_back(j);
  }
  // reconstruct (sie.py:332-346): IN = traces in the down layout, full-volume output
  for (int l = 0; l < L; ++l) {
    OJob j = blank_job(l);
    j.vol = 1;
    j.nout = -1;
    if (l >= 1) {
      j.pan[0][0] = Ref{0, segD(c, l - 1, 0)};
      j.pan[1][0] = Ref{0, segD(c, l - 1, 1)};
    }
    if (l <= L - 2) {
      j.pan[2][0] = Ref{0, segD(c, l, 0)};
      j.pan[3][0] = Ref{0, segD(c, l, 1)};
    }
    c->recon.jobs.push_back(j);
  }
  int rc = 0;
  rc |= finalize_stage(c, c->newton);
  rc |= finalize_stage(c, c->op);
  rc |= finalize_stage(c, c->refl);
  rc |= finalize_stage(c, c->recon);
  for (int I = 1; I < nI; ++I) rc |= finalize_stage(c, c->sdown[I]);
  for (int I = 0; I <= nI - 2; ++I) rc |= finalize_stage(c, c->sup[I]);
  return rc ? PT_CUDA_ERROR : 0;
}

// inner programs over cells (nested.py:125-153 -> sie.py:203-326); vec ids 0 IN, 1 OUT, 2 AUX; seg units of w
static int build_inner(pt_ctx* c) {
  const int Lc = c->Lc, nI = Lc - 1;
  auto D = [&](int I, int s) { return 2 * I + s; };
  auto U = [&](int I, int s) { return 2 * nI + 2 * I + s; };
  auto item = [&](int cell, int row) {
    IItem it;
    std::memset(&it, 0, sizeof(it));
    it.cell = cell;
    it.row = row;
    for (int s = 0; s < 4; ++s) it.pan[s][0] = it.pan[s][1] = NOREF;
    it.dst = it.add[0] = it.add[1] = it.sub[0] = it.sub[1] = it.rev = NOREF;
    it.flags = 0;
    return it;
  };
  std::vector<IItem> items;
  std::vector<int> oph, pph;
  long long opb = 0, preb = 0;
  auto count = [&](const IItem& it, long long& acc) {
    if (it.cell < 0) return;
    for (int s = 0; s < 4; ++s)
      if (it.pan[s][0].vec >= 0) ++acc;
  };
  // ---- OP (sie.py:203-228): one phase.  The full traces d + p of the reference are summed
  // element-wise while the panels are gathered (pan[s][1]), and "- (d + p)" is sub0 + sub1.
  oph.push_back((int)items.size());
  for (int cc = 0; cc < Lc; ++cc) {
    const bool top = cc >= 1, bot = cc <= Lc - 2;
    const int ib = cc, it = cc - 1;
    if (bot) {
      for (int s = 0; s < 2; ++s) {
        IItem x = item(cc, 2 + s);
        if (top) {  // v0, v1 = d + p above
          for (int k = 0; k < 2; ++k) {
            x.pan[k][0] = Ref{0, D(ib - 1, k)};
            x.pan[k][1] = Ref{0, U(ib - 1, k)};
          }
        }
        x.pan[2][0] = Ref{0, U(ib, 0)};
        x.pan[3][0] = Ref{0, U(ib, 1)};
        x.dst = Ref{1, D(ib, s)};
        x.sub[0] = Ref{0, D(ib, s)};        // wb[0] - (d + p) ; wb[1] - d
        if (s == 0) x.sub[1] = Ref{0, U(ib, 0)};
        count(x, opb);
        items.push_back(x);
      }
    }
    if (top) {
      for (int s = 0; s < 2; ++s) {
        IItem x = item(cc, s);
        x.pan[0][0] = Ref{0, D(it, 0)};
        x.pan[1][0] = Ref{0, D(it, 1)};
        if (bot) {  // vn, vnp = p + d below
          for (int k = 0; k < 2; ++k) {
            x.pan[2 + k][0] = Ref{0, U(ib, k)};
            x.pan[2 + k][1] = Ref{0, D(ib, k)};
          }
        }
        x.dst = Ref{1, U(it, s)};
        x.sub[0] = Ref{0, U(it, s)};        // wt[0] - p ; wt[1] - (d + p)
        if (s == 1) x.sub[1] = Ref{0, D(it, 1)};
        count(x, opb);
        items.push_back(x);
      }
    }
  }
  oph.push_back((int)items.size());
  // ---- PRE (GS, sie.py:322-326) in 2 nI - 1 phases: the down sweep (phase k computes y_down[k];
  // phase 1 also y_down[0] = -v_down[0]), each reflection as soon as its y_down panels exist, and
  // the up sweep.  The combinations s = p - refl and y_up[nI-1] = -s[nI-1] are folded into the
  // reflection items (modes 1 and 2; exact: -(p - t) == t - p in IEEE arithmetic).  Items of
  // phase 1 read y_down[0] as the negated v_down[0] (also exact).
  std::vector<std::vector<IItem>> P(2 * nI + 1);  // P[1 .. 2nI-1]
  for (int s = 0; s < 2 && nI > 0; ++s) {          // y_down[0] = -v_down[0]
    IItem x = item(-1, 0);
    x.dst = Ref{1, D(0, s)};
    x.sub[0] = Ref{0, D(0, s)};
    P[1].push_back(x);
  }
  for (int I = 1; I < nI; ++I)
    for (int s = 0; s < 2; ++s) {
      IItem x = item(I, 2 + s);
      x.pan[0][0] = Ref{1, D(I - 1, 0)};
      x.pan[1][0] = Ref{1, D(I - 1, 1)};
      x.dst = Ref{1, D(I, s)};
      x.sub[0] = Ref{0, D(I, s)};
      count(x, preb);
      P[I].push_back(x);
    }
  for (int I = 0; I < nI; ++I)
    for (int s = 0; s < 2; ++s) {
      IItem x = item(I + 1, s);
      x.pan[0][0] = Ref{1, D(I, 0)};
      x.pan[1][0] = Ref{1, D(I, 1)};
      if (I <= nI - 2) {
        x.pan[2][0] = Ref{1, D(I + 1, 0)};
        x.pan[3][0] = Ref{1, D(I + 1, 1)};
      }
      if (s == 1) x.sub[0] = Ref{1, D(I, 1)};
      x.rev = Ref{0, U(I, s)};
      if (I == nI - 1) {
        x.dst = Ref{1, U(I, s)};  // y_up[nI-1] = -(p - refl) = refl - p
        x.flags |= 2 << 8;
      } else {
        x.dst = Ref{2, U(I, s)};  // s = p - refl
        x.flags |= 1 << 8;
      }
      count(x, preb);
      const int ph = I <= nI - 2 ? I + 2 : nI;
      if (ph == 1) {  // nI == 1: y_down[0] is produced in this same phase; read -v_down[0]
        for (int k = 0; k < 2; ++k)
          if (x.pan[k][0].vec == 1 && x.pan[k][0].seg == D(0, k)) {
            x.pan[k][0].vec = 0;
            x.flags |= 1 << k;
          }
        if (x.sub[0].vec == 1 && x.sub[0].seg == D(0, 1)) {  // - (-v) == + v
          x.add[0] = Ref{0, D(0, 1)};
          x.sub[0] = NOREF;
        }
      }
      P[ph].push_back(x);
    }
  for (int I = nI - 2; I >= 0; --I)
    for (int s = 0; s < 2; ++s) {
      IItem x = item(I + 1, s);
      x.pan[2][0] = Ref{1, U(I + 1, 0)};
      x.pan[3][0] = Ref{1, U(I + 1, 1)};
      x.dst = Ref{1, U(I, s)};
      x.sub[0] = Ref{2, U(I, s)};
      count(x, preb);
      P[nI + (nI - 1 - I)].push_back(x);
    }
  // phase 1: the down-sweep items read y_down[0] = -v_down[0] directly
  for (IItem& x : P[nI > 0 ? 1 : 0])
    if (x.cell >= 0)
      for (int k = 0; k < 2; ++k)
        if (x.pan[k][0].vec == 1 && x.pan[k][0].seg == D(0, k)) {
          x.pan[k][0].vec = 0;
          x.flags |= 1 << k;
        }
  pph.push_back((int)items.size());
  for (int ph = 1; ph <= 2 * nI - 1; ++ph) {
    for (const IItem& x : P[ph]) items.push_back(x);
    pph.push_back((int)items.size());
  }
  for (IItem& x : items) {
    int ns = 0;
    if (x.cell >= 0)
      for (int k = 0; k < 4; ++k) ns += x.pan[k][0].vec >= 0;
    x.wgt = ns > 0 ? ns : 1;
  }
  c->op_nph = (int)oph.size() - 1;
  c->pre_nph = (int)pph.size() - 1;
  c->op_blocks = opb;
  c->pre_blocks = preb;
  c->nitems = (int)items.size();
  if (nI == 0) return 0;
  if (upload(&c->items_d, items.data(), items.size())) return PT_CUDA_ERROR;
  if (upload(&c->op_ph_d, oph.data(), oph.size())) return PT_CUDA_ERROR;
  if (upload(&c->pre_ph_d, pph.data(), pph.size())) return PT_CUDA_ERROR;
  // ---- PRE, scan form.  The down sweep y_I = T_I y_{I-1} - v_I (sie.py:272-283 on the cells; T_I the 2 x 2 block
  // matrix of cell I's Green blocks (rows n, n+1; slots v0, v1)) is a linear recurrence: with the products
  // T^(2)_I = T_I T_{I-1}, T^(4)_I = T^(2)_I T^(2)_{I-2}, ... (create_impl) every y_I follows in ceil(log2 nI)
  // data-parallel levels  d_I <- T^(st)_I d_{I-st} + d_I  (st = 1, 2, 4, ...; d_I starts as -v_I) instead of
  // nI - 1 dependent phases; likewise the up sweep (sie.py:285-296) with U_I (rows 0, 1; slots vn, vnp of cell
  // I + 1).  Same linear map as the sequential program (rounding order aside), 2 levels + 1 phases per
  // application instead of 2 nI - 1: used where a stage is one job (the sequential outer sweeps), whose phases are
  // latency-bound.  An index's value ping-pongs between its OUT segment and a spare AUX segment so that no level
  // writes what another item of the level reads; the last update of every index lands in OUT.
  if (c->scan_levels > 0 && nI >= 3) {
    std::vector<IItem> px(items.begin(), items.begin() + oph.back());  // the op program, unchanged
    std::vector<int> ph;
    int nlev = 0;
    while ((1 << nlev) < nI) ++nlev;  // strides 1 .. 2^(nlev-1)
    if (nlev - 1 > c->scan_levels) return 0;
    struct Cur {
      Ref r[2];
      bool neg;
    };
    auto nupd = [](int dist) {  // updates of an index at distance dist >= 1 from the chain start
      int n = 0;
      while ((1 << n) <= dist) ++n;
      return n;
    };
    // one chain: down (dir 0: index I, predecessor I - st, start I = 0) or up (dir 1: predecessor I + st, start nI - 1)
    auto chain = [&](int dir, std::vector<Cur>& cur) {
      std::vector<int> done(nI, 0);
      for (int lv = 0; lv < nlev; ++lv) {
        const int st = 1 << lv;
        std::vector<Cur> nxt = cur;
        for (int I = 0; I < nI; ++I) {
          const int dist = dir == 0 ? I : nI - 1 - I;
          if (dist < st) continue;
          const int Pd = dir == 0 ? I - st : I + st;
          const int cell = dir == 0 ? I : I + 1;
          const int n = nupd(dist), k = ++done[I];
          for (int sb = 0; sb < 2; ++sb) {
            IItem x = item(cell, lv == 0 ? (dir == 0 ? 2 + sb : sb) : 4 + (lv - 1) * 2 + sb);
            for (int kk = 0; kk < 2; ++kk) {
              const int slot = dir == 0 ? kk : 2 + kk;
              x.pan[slot][0] = cur[Pd].r[kk];
              if (cur[Pd].neg) x.flags |= 1 << slot;
            }
            if (cur[I].neg) x.sub[0] = cur[I].r[sb];
            else x.add[0] = cur[I].r[sb];
            const bool to_out = ((n - k) & 1) == 0;
            x.dst = to_out ? Ref{1, dir == 0 ? D(I, sb) : U(I, sb)} : Ref{2, D(I, sb)};
            nxt[I].r[sb] = x.dst;
            px.push_back(x);
          }
          nxt[I].neg = false;
        }
        cur = nxt;
        ph.push_back((int)px.size());
      }
    };
    ph.push_back((int)px.size());
    // phase 0 of the down chain also holds y_down[0] = -v_down[0]
    for (int sb = 0; sb < 2; ++sb) {
      IItem x = item(-1, 0);
      x.dst = Ref{1, D(0, sb)};
      x.sub[0] = Ref{0, D(0, sb)};
      px.push_back(x);
    }
    {
      std::vector<Cur> cur(nI);
      for (int I = 0; I < nI; ++I) cur[I] = Cur{{Ref{0, D(I, 0)}, Ref{0, D(I, 1)}}, true};  // d_I = -v_I (IN)
      chain(0, cur);
    }
    // reflections (sie.py:298-308) in one phase on the finished y_down; s = p - refl -> AUX, y_up[nI-1] -> OUT
    for (int I = 0; I < nI; ++I)
      for (int sb = 0; sb < 2; ++sb) {
        IItem x = item(I + 1, sb);
        x.pan[0][0] = Ref{1, D(I, 0)};
        x.pan[1][0] = Ref{1, D(I, 1)};
        if (I <= nI - 2) {
          x.pan[2][0] = Ref{1, D(I + 1, 0)};
          x.pan[3][0] = Ref{1, D(I + 1, 1)};
        }
        if (sb == 1) x.sub[0] = Ref{1, D(I, 1)};
        x.rev = Ref{0, U(I, sb)};
        if (I == nI - 1) {
          x.dst = Ref{1, U(I, sb)};
          x.flags |= 2 << 8;
        } else {
          x.dst = Ref{2, U(I, sb)};
          x.flags |= 1 << 8;
        }
        px.push_back(x);
      }
    ph.push_back((int)px.size());
    {
      std::vector<Cur> cur(nI);
      for (int I = 0; I < nI; ++I) cur[I] = Cur{{Ref{2, U(I, 0)}, Ref{2, U(I, 1)}}, true};  // e_I = -s_I (AUX)
      cur[nI - 1] = Cur{{Ref{1, U(nI - 1, 0)}, Ref{1, U(nI - 1, 1)}}, false};               // y_up[nI-1] (OUT)
      chain(1, cur);
    }
    for (IItem& x : px) {
      int ns = 0;
      if (x.cell >= 0)
        for (int k = 0; k < 4; ++k) ns += x.pan[k][0].vec >= 0;
      x.wgt = ns > 0 ? ns : 1;
    }
    // phase offsets: ph[0] = first pre item; the y_down[0] items belong to the first level's phase
    std::vector<int> pph2;
    pph2.push_back(ph[0]);
    for (size_t i = 1; i < ph.size(); ++i) pph2.push_back(ph[i]);
    c->pre_nph_px = (int)pph2.size() - 1;
    c->nitems_px = (int)px.size();
    if (upload(&c->items_px_d, px.data(), px.size())) return PT_CUDA_ERROR;
    if (upload(&c->pre_ph_px_d, pph2.data(), pph2.size())) return PT_CUDA_ERROR;
  }
  return 0;
}

// ------------------------------------------------------------------ scratch

static int ensure_scratch(pt_ctx* c, int R, int capO) {
  const int Jmax = std::max(std::max(2 * c->L - 2, c->L), 1);
  if (R <= c->capR && capO <= c->capO) return 0;
  R = std::max(R, c->capR);
  capO = std::max(capO, c->capO);
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  for (void* p : {(void*)c->V, (void*)c->Bv, (void*)c->Bp, (void*)c->T1, (void*)c->AX, (void*)c->X, (void*)c->TR,
                  (void*)c->ipart,
                  (void*)c->P, (void*)c->smp, (void*)c->tables, (void*)c->tables_f, (void*)c->trc, (void*)c->iscr,
                  (void*)c->hess, (void*)c->iters, (void*)c->istate, (void*)c->ibeta0, (void*)c->rmap_d, (void*)c->dscal,
                  (void*)c->hout, (void*)c->ybuf})
    F(p);
  if (c->hrmap) cudaFreeHost(c->hrmap);
  if (c->hhout) cudaFreeHost(c->hhout);
  if (c->hdscal) cudaFreeHost(c->hdscal);
  if (c->hy) cudaFreeHost(c->hy);
  const long long nO = std::max(4LL * c->nI * c->wx, 1LL);
  c->nO = nO;
  CK(cudaMalloc(&c->V, sizeof(double2) * (size_t)R * (capO + 1) * nO));
  for (double2** p : {&c->Bv, &c->Bp, &c->T1, &c->AX, &c->X, &c->TR}) CK(cudaMalloc(p, sizeof(double2) * (size_t)R * nO));
  CK(cudaMalloc(&c->P, sizeof(double2) * (size_t)Jmax * 4 * R * c->wx));
  CK(cudaMalloc(&c->smp, sizeof(double2) * (size_t)Jmax * 4 * R * c->wx));
  CK(cudaMalloc(&c->tables, sizeof(double2) * (size_t)Jmax * c->Lc * 4 * R * c->wmax));
  CK(cudaMalloc(&c->tables_f, sizeof(double2) * (size_t)Jmax * c->Lc * 4 * R * c->wmax));
  CK(cudaMalloc(&c->trc, sizeof(double2) * (size_t)Jmax * R * std::max(c->Lc - 1, 1) * 2 * c->wmax));
  c->inmax = 4LL * std::max(c->Lc - 1, 1) * c->wmax;
  c->iscr_stride = (long long)(c->inner_cap + 5) * c->inmax;
  // instances padded to whole n-tiles of 8 (the item-program kernel's RHS-minor layout uses the same buffer)
  const int Rp = (R + 7) / 8 * 8;
  CK(cudaMalloc(&c->iscr, sizeof(double2) * (size_t)Jmax * Rp * c->iscr_stride));
  c->ipart_items = inner_items_part_items(c->num_sms, Jmax, Rp);
  CK(cudaMalloc(&c->ipart, sizeof(double2) * (size_t)3 * c->ipart_items * (c->inner_cap + 2) * 8));
  c->hstride = (long long)(c->inner_cap + 1) * c->inner_cap + (c->inner_cap + 1) + 2 * c->inner_cap;
  CK(cudaMalloc(&c->hess, sizeof(double2) * (size_t)Jmax * R * c->hstride));
  CK(cudaMalloc(&c->iters, sizeof(int) * (size_t)Jmax * R));
  CK(cudaMalloc(&c->istate, sizeof(int) * (size_t)Jmax * R));
  CK(cudaMalloc(&c->ibeta0, sizeof(double) * (size_t)Jmax * R));
  CK(cudaMalloc(&c->rmap_d, sizeof(int) * R));
  CK(cudaMalloc(&c->dscal, sizeof(double) * 2 * R));
  CK(cudaMalloc(&c->hout, sizeof(double2) * (size_t)R * (capO + 2)));
  CK(cudaMalloc(&c->ybuf, sizeof(double2) * (size_t)R * (capO + 1)));
  CK(cudaMallocHost(&c->hrmap, sizeof(int) * R * PT_RMAP_SLOTS));
  CK(cudaMallocHost(&c->hhout, sizeof(double2) * (size_t)R * (capO + 2)));
  CK(cudaMallocHost(&c->hdscal, sizeof(double) * 2 * R));
  CK(cudaMallocHost(&c->hy, sizeof(double2) * (size_t)R * (capO + 1)));
  c->capR = R;
  c->capO = capO;
  c->gen++;
  return 0;
}

static int ensure_z(pt_ctx* c, long long z) {
  if (z <= c->zcap) return 0;
  if (c->Z) cudaFree(c->Z);
  CK(cudaMalloc(&c->Z, sizeof(double2) * (size_t)z));
  c->zcap = z;
  c->gen++;
  return 0;
}

// K1 launch geometry for a stage: NC columns per CTA, CM column-CTAs per half-chain (multicast
// group); a task = (cell, CM*NC columns of one layer) = one cluster of 2*CM CTAs.
static void k1_policy(pt_ctx* c, const std::vector<int>& ncols_per_group, int* nc_out, int* cm_out) {
  int cm = 1;
  if (const char* e = std::getenv("PT_K1_CM")) cm = std::max(1, std::min(8, atoi(e)));
  int nc = 0;
  if (const char* e = std::getenv("PT_K1_NC")) nc = atoi(e);
  if (nc != 1 && nc != 2 && nc != 4 && nc != 8) {
    // Minimise (waves of CTA pairs) x (relative cost of one launch wave at this NC): one K1 CTA per
    // SM, so a stage with more CTAs than SMs runs in several waves.  Relative per-wave costs were
    // measured on the B200 for w = 70 (tools/k1_probe.py): NC=1 1.0, 2 1.45, 4 2.15, 8 2.5.
    nc = 1;
    double best = 1e30;
    for (int cand : {1, 2, 4, 8}) {
      if (cand * c->wmax > 640 && cand > 1) continue;  // keep the partial sums next to the ring
      long long tasks = 0;
      for (int n : ncols_per_group) tasks += (long long)c->Lc * ((n + cand * cm - 1) / (cand * cm));
      const double cost = cand == 1 ? 1.0 : cand == 2 ? 1.45 : cand == 4 ? 2.15 : 2.5;
      const long long waves = (2LL * cm * tasks + c->num_sms - 1) / c->num_sms;
      const double t = (double)waves * cost;
      if (t < best - 1e-9) {
        best = t;
        nc = cand;
      }
    }
  }
  while (cm > 1 && c->ns % cm) --cm;
  *nc_out = nc;
  *cm_out = cm;
}

static Stage::Tasks* stage_tasks(pt_ctx* c, Stage& S, int Ract) {
  auto itr = S.tasks.find(Ract);
  if (itr != S.tasks.end()) return &itr->second;
  Stage::Tasks T;
  std::vector<int> ncols;
  for (size_t g = 0; g < S.lgrp.size(); ++g) {
    const int b = S.lgrp[g].second;
    const int e = g + 1 < S.lgrp.size() ? S.lgrp[g + 1].second : (int)S.ljobs.size();
    ncols.push_back((e - b) * Ract);
  }
  int nc = 1, cm = 1;
  k1_policy(c, ncols, &nc, &cm);
  T.nc = nc;
  T.cm = cm;
  std::vector<K1Task> v;
  long long z = 0;
  for (size_t g = 0; g < S.lgrp.size(); ++g) {
    const int l = S.lgrp[g].first, b = S.lgrp[g].second;
    const int n = ncols[g];
    // cell-major: the column groups of one cell are neighbours in the launch order, so the CTA pairs that stream
    // the same factor blocks run together and share them in L2 (PT_K1_COLMAJOR: column-group-major, round 1's order)
    static const bool colmajor = std::getenv("PT_K1_COLMAJOR") != nullptr;
    const int ngq = (n + nc * cm - 1) / (nc * cm);
    for (int it = 0; it < ngq * c->Lc; ++it) {
        const int cc = colmajor ? it % c->Lc : it / ngq;
        const int q0 = (colmajor ? it / c->Lc : it % ngq) * nc * cm;
        const CellInfo& ci = c->cel[l * c->Lc + cc];
        K1Task t;
        t.cell = l * c->Lc + cc;
        t.jb = b;
        t.q0 = q0;
        t.nq = std::min(nc * cm, n - q0);
        t.zoff = z;
        z += (long long)cm * ci.wzc * ci.w * nc;
        T.bytes += 32.0 * ci.wzc * (double)ci.w * ci.w * t.nq;
        T.hbytes += 16.0 * ci.wzc * (double)ci.w * ci.w;
        v.push_back(t);
      }
  }
  T.n = (int)v.size();
  T.zsize = z;
  if (upload(&T.d, v.data(), v.size())) return nullptr;
  c->gen++;
  auto res = S.tasks.emplace(Ract, T);
  return &res.first->second;
}

// ------------------------------------------------------------------ stage execution

struct SolveIO {
  const double2* f;
  long long f_stride;
  double2* u;
  long long u_stride;
  double inner_ktol;
  int inner_max_iter;
};

static int grid_for(long long n) {
  long long b = (n + 255) / 256;
  return (int)std::max(1LL, std::min(b, 148LL * 16));
}

static InnerParams inner_params(pt_ctx* c, Stage& S, int Ract, const SolveIO& io) {
  InnerParams ip;
  std::memset(&ip, 0, sizeof(ip));
  ip.cells = c->cel_d;
  ip.layers = c->lay_d;
  ip.jobs = S.jobs_d;
  ip.stage_jobs = S.stage_jobs_d;
  ip.green = c->green_d;
  static const bool no_dense = std::getenv("PT_NO_DENSE") != nullptr;
  ip.dense = no_dense ? nullptr : c->dense_d;
  ip.items = c->items_d;
  ip.op_ph = c->op_ph_d;
  ip.op_nph = c->op_nph;
  ip.pre_ph = c->pre_ph_d;
  ip.pre_nph = c->pre_nph;
  ip.R = Ract;
  ip.Lc = c->Lc;
  ip.wmax = c->wmax;
  ip.cap = c->inner_cap;
  ip.max_iter = io.inner_max_iter;
  ip.ktol = io.inner_ktol;
  ip.tables = c->tables;
  ip.tr = c->trc;
  ip.scratch = c->iscr;
  ip.inst_stride = c->iscr_stride;
  ip.nmax = c->inmax;
  ip.hess = c->hess;
  ip.hstride = c->hstride;
  ip.iters = c->iters;
  ip.state = c->istate;
  ip.beta0 = c->ibeta0;
  ip.err = c->err_d;
  ip.counters = c->cnt_d;
  ip.hist = c->hist_d;
  ip.op_blocks = c->op_blocks;
  ip.pre_blocks = c->pre_blocks;
  ip.tprof = std::getenv("PT_INNER_TPROF") != nullptr;
  ip.nitems = c->nitems;
  ip.items_px = c->items_px_d;
  ip.pre_ph_px = c->pre_ph_px_d;
  ip.pre_nph_px = c->pre_nph_px;
  ip.nitems_px = c->nitems_px;
  ip.mg = inner_mg(c->wmax);
  ip.tring = inner_tring(c->wmax, ip.nitems);
  static const bool arn_slow = std::getenv("PT_ARN_SLOW") != nullptr;
  ip.arn_fast = !arn_slow;
  ip.coop_sms = c->coop_sms;
  ip.part = c->ipart;
  ip.part_items = c->ipart_items;
  ip.ii_dbg = std::getenv("PT_II_DBG") ? atoi(std::getenv("PT_II_DBG")) : 0;
  static const int tilecost = std::getenv("PT_II_TILECOST") ? atoi(std::getenv("PT_II_TILECOST")) : 0;
  ip.ii_tilecost = tilecost;
  ip.ii_trace = std::getenv("PT_II_TRACE") ? atoi(std::getenv("PT_II_TRACE")) : 0;
  static const bool unit_major = std::getenv("PT_UNIT_MAJOR") != nullptr;
  ip.unit_major = unit_major;
  // opt-in (PT_TPREFETCH=1): measured slower (cfg5 1 source 1328 vs 1217 ms; the prefetch delays each CTA's
  // arrival at the grid barrier more than it saves after it)
  static const bool tprefetch = std::getenv("PT_TPREFETCH") != nullptr;
  ip.tprefetch = tprefetch;
  static const bool no_sstep = std::getenv("PT_NO_SSTEP") != nullptr;
  ip.sstep = !no_sstep && c->dense_cnt >= 4 && c->dense_d;
  if (ip.tring < 4 * ip.mg) ip.mg = 1;  // a group's (slot, row tile) tiles must fit in the ring together
  return ip;
}

// Executed work per launch class of a stage (per active RHS) and the operator bytes it streams:
// pass-0 product 8 Mp (used slots x nk4) per (job, cell); sampled response 8 (kept rows x outputs) (slots x w) per
// (job, cell); inner GMRES: the Green blocks of the stage's layers (16 blocks of w^2 per cell) -- its flops are
// the device's TouchCounter total x 8, added at the end of the solve.
static void stage_work(pt_ctx* c, Stage& S) {
  if (S.work_ok) return;
  S.work_ok = true;
  std::vector<char> seen(c->L, 0);
  for (size_t g = 0; g < S.lgrp.size(); ++g) {
    const int l = S.lgrp[g].first, b = S.lgrp[g].second;
    const int e = g + 1 < S.lgrp.size() ? S.lgrp[g + 1].second : (int)S.ljobs.size();
    int used = 0;
    for (int jj = b; jj < e; ++jj)
      for (int sl = 0; sl < 4; ++sl) used |= (S.jobs[S.ljobs[jj]].pan[sl][0].vec >= 0) << sl;
    const int nsl = __builtin_popcount(used);
    for (int cc = 0; cc < c->Lc; ++cc) {
      const CellInfo& ci = c->cel[l * c->Lc + cc];
      // executed rows: the Newton-table rows and, per job, the sample rows of the output rows it samples (whole
      // tiles of the others are skipped); operator bytes: the rows some job of the group needs
      const int nk = ci.hi - ci.lo, nk4 = (nk + 3) & ~3;
      int oall = 0;
      double rows_j = 0;
      for (int jj = b; jj < e; ++jj) {
        const OJob& jo = S.jobs[S.ljobs[jj]];
        int om = 0;
        for (int o = 0; o < jo.nout; ++o)
          om |= 1 << (jo.orow[o] == 0 ? 0 : (jo.orow[o] == 1 ? 1 : (jo.orow[o] == c->lay[l].n ? 2 : 3)));
        oall |= om;
        rows_j += q0_tab8(ci.w) + (double)__builtin_popcount(om) * q0_nk8(nk);
      }
      S.p0_fpr += 8.0 * rows_j * nsl * nk4;
      S.p0_bytes += 16.0 * (q0_tab8(ci.w) + (double)__builtin_popcount(oall) * q0_nk8(nk)) * nsl * nk4;
      if (!seen[l]) S.in_bytes += 16.0 * 16.0 * ci.w * ci.w;
    }
    seen[l] = 1;
  }
  for (const OJob& jb : S.jobs) {
    if (jb.nout <= 0) continue;
    for (int cc = 0; cc < c->Lc; ++cc) {
      const CellInfo& ci = c->cel[jb.layer * c->Lc + cc];
      const double rows = (double)(ci.hi - ci.lo) * jb.nout;
      const double K = (double)((ci.has_bot ? 4 : 2) - (ci.has_top ? 0 : 2)) * ci.w;
      S.gs_fpr += 8.0 * rows * K;
      S.gs_bytes += 16.0 * rows * K;
    }
  }
}

static int run_stage(pt_ctx* c, Stage& S, VecTab tab, int Ract, const SolveIO& io) {
  c->cur_tag = S.name;
  const int J = (int)S.jobs.size();
  if (J == 0 || Ract == 0) return 0;
  Stage::Tasks* T = stage_tasks(c, S, Ract);
  if (!T) return PT_CUDA_ERROR;
  if (ensure_z(c, T->zsize)) return PT_CUDA_ERROR;
  stage_work(c, S);
  // optionally one cooperative launch for a whole sample-only stage without volume source (gather, pass-0
  // product, inner GMRES, sampled response, combine); falls back to the launch sequence below
  {
    // opt-in (PT_FUSE=1): measured slower than the separate launches on cfg2 (one 8-warp CTA per SM hides
    // less latency in the pass-0 / sampled-response products than their own many-CTA grids)
    static const bool no_fuse = std::getenv("PT_FUSE") == nullptr;
    static const bool no_q0e = std::getenv("PT_NO_Q0") != nullptr, no_gsmpe = std::getenv("PT_NO_GSMP") != nullptr;
    static const bool no_dense = std::getenv("PT_NO_DENSE") != nullptr, no_coop = std::getenv("PT_NO_COOP") != nullptr;
    if (!no_fuse && !no_q0e && !no_gsmpe && !no_dense && !no_coop && c->Lc > 1 && c->gsmp_d && c->q0_d &&
        c->dense_d && S.samples_only && S.no_volume && S.any_panel && S.grp_d) {
      InnerParams ip = inner_params(c, S, Ract, io);
      ip.fused = 1;
      ip.tab = tab;
      ip.rmap = c->rmap_d;
      ip.wx = c->wx;
      ip.ngl = (int)S.lgrp.size();
      int maxj = 0;
      for (size_t i = 0; i < S.lgrp.size(); ++i) {
        const int e = i + 1 < S.lgrp.size() ? S.lgrp[i + 1].second : (int)S.ljobs.size();
        maxj = std::max(maxj, e - S.lgrp[i].second);
      }
      ip.maxj = maxj;
      ip.kmax = c->wzcmax;
      ip.P = c->P;
      ip.smp = c->smp;
      ip.q0 = c->q0_d;
      ip.gsmp = c->gsmp_d;
      ip.grp = S.grp_d;
      ip.ljobs = S.ljobs_d;
      c->cur_tag = S.name;
      cudaError_t e;
      {
        LaunchScope ls(c, 1);
        e = inner_coop_launch(ip, J, c->st);
      }
      if (e == cudaSuccess) {
        if (ip.tprof) inner_tprof_dump(S.name);
        c->layer_solves += (long long)J * Ract;
        if (!c->asm_touch.empty())
          for (const OJob& jb : S.jobs) c->touch_extra += c->asm_touch[jb.layer] * Ract;
        return 0;
      }
      if (e != cudaErrorNotSupported) CK(e);
      cudaGetLastError();
    }
  }
  // one-pass layer solve: samples = pass-0 samples + sampled trace responses (linearity)
  static const bool no_gsmp = std::getenv("PT_NO_GSMP") != nullptr;
  const bool gpath = c->Lc > 1 && c->gsmp_d && S.samples_only && !no_gsmp;
  static const bool no_q0 = std::getenv("PT_NO_Q0") != nullptr;
  const bool qpath = gpath && c->q0_d && S.no_volume && S.any_panel && S.grp_d && !no_q0;
  // RECON: first pass by linearity = Newton tables of f (saved by the NEWTON stage) + pass-0 product of
  // the trace panels (the jobs of both stages are the L layers in order, same RHS set)
  static const bool no_reuse = std::getenv("PT_NO_REUSE") != nullptr;
  const bool rpath = &S == &c->recon && c->tables_f_ok && c->q0_d && S.any_panel && S.grp_d && !no_reuse &&
                     Ract == c->tables_f_R;
  // opt-in (PT_FUSE_GLUE=1): gather fused into the pass-0 product where nothing else needs P; measured
  // slower on cfg2 (the panel refs are re-read in the inner loops)
  static const bool no_fuse_glue = std::getenv("PT_FUSE_GLUE") == nullptr;
  const bool direct_b = qpath && !no_fuse_glue;   // pass-0 reads the panels straight from the vectors
  // the sampled response writes the combined outputs (k_combine folded in; PT_NO_FUSE_COMB keeps it apart)
  static const bool no_fuse_comb = std::getenv("PT_NO_FUSE_COMB") != nullptr;
  const bool fuse_comb = gpath && (!no_fuse_glue || !no_fuse_comb);
  if (S.any_panel && !direct_b) {
    LaunchScope ls(c, 2);
    k_gather_panels<<<grid_for((long long)J * 4 * Ract * c->wx), 256, 0, c->st>>>(S.jobs_d, J, tab, c->rmap_d, Ract,
                                                                                    c->wx, c->P);
    CK(cudaGetLastError());
  }
  K1Params kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.cells = c->cel_d;
  kp.layers = c->lay_d;
  kp.jobs = S.jobs_d;
  kp.ljobs = S.ljobs_d;
  kp.tasks = T->d;
  kp.sinv = c->sinv_d;
  kp.lz = c->lz_d;
  kp.uz = c->uz_d;
  kp.R = Ract;
  kp.npml = c->npml;
  kp.wx = c->wx;
  kp.Lc = c->Lc;
  kp.wmax = c->wmax;
  kp.slot_bytes = c->slot_bytes;
  kp.ns = c->ns;
  kp.cm = T->cm;
  kp.f = io.f;
  kp.f_stride = io.f_stride;
  kp.P = c->P;
  kp.tr = c->trc;
  kp.tables = c->tables;
  kp.smp = c->smp;
  kp.u = io.u;
  kp.u_stride = io.u_stride;
  kp.Z = c->Z;
  static long long* tprof_d = nullptr;
  static bool tprof_on = std::getenv("PT_K1_TPROF") != nullptr;
  if (tprof_on && !tprof_d) cudaMalloc(&tprof_d, 6 * sizeof(long long));
  kp.tprof = tprof_on ? tprof_d : nullptr;
  kp.dbg = std::getenv("PT_K1_DBG") ? atoi(std::getenv("PT_K1_DBG")) : 0;
  // volume sources/outputs are indexed by the real RHS id: pre-offset through rmap on the host is not
  // possible per column, so stage buffers use compact q and f/u use q as well (callers compact f/u).
  kp.s0 = gpath ? 1 : 0;
  if (c->Lc > 1) {
    kp.pass = 0;
    // pass-0 products also write the inner rhs (rhs_pol) into the inner scratch: the inner kernel skips its
    // gather pass and one grid barrier (dense cooperative path; PT_NO_RHS_OUT keeps the gather)
    static const bool no_rhs_out = std::getenv("PT_NO_RHS_OUT") != nullptr;
    const RhsOut ro{c->iscr, c->iscr_stride, (long long)(c->inner_cap + 1) * c->inmax};
    const bool rhs_out = !no_rhs_out && c->dense_d && !c->lu_d && (rpath || qpath);
    if (rpath || qpath) {
      c->cls_flops[4] += S.p0_fpr * Ract;
      c->cls_bytes[4] += S.p0_bytes;
    } else {
      c->cls_flops[0] += T->bytes / 4.0;  // one complex MAC (8 flops) per S^-1 element per column
      c->cls_bytes[0] += T->hbytes;
    }
    if (rpath) {
      LaunchScope ls(c, 4);
      CK(cudaMemcpyAsync(c->tables, c->tables_f, sizeof(double2) * (size_t)J * c->Lc * 4 * Ract * c->wmax,
                         cudaMemcpyDeviceToDevice, c->st));
      CK(pass0_launch(S.grp_d, (int)S.lgrp.size(), S.ljobs_d, S.jobs_d, c->cel_d, c->lay_d, c->q0_d, c->P, c->tables,
                      c->smp, Ract, c->Lc, c->wx, c->wmax, c->wzcmax, 1, c->st, 1, nullptr, nullptr,
                      rhs_out ? &ro : nullptr));
    } else if (qpath) {  // first pass as one dense product with the offline pass-0 operators (no volume source)
      LaunchScope ls(c, 4);
      int maxj = 0;
      for (size_t i = 0; i < S.lgrp.size(); ++i) {
        const int e = i + 1 < S.lgrp.size() ? S.lgrp[i + 1].second : (int)S.ljobs.size();
        maxj = std::max(maxj, e - S.lgrp[i].second);
      }
      CK(pass0_launch(S.grp_d, (int)S.lgrp.size(), S.ljobs_d, S.jobs_d, c->cel_d, c->lay_d, c->q0_d, c->P, c->tables,
                      c->smp, Ract, c->Lc, c->wx, c->wmax, c->wzcmax, maxj, c->st, 0, direct_b ? &tab : nullptr,
                      c->rmap_d, rhs_out ? &ro : nullptr));
    } else {
      LaunchScope ls(c, 0);
      // NEWTON (sie.py:175-188): a layer's solve of a source that is zero inside the layer is zero -- point and
      // surface sources touch one layer of L.  Flag the (layer, RHS) slabs that hold a nonzero; K1 tasks whose
      // columns are all unflagged write zero tables / samples and exit (PT_NO_ZSKIP solves them all).
      static const bool no_zskip = std::getenv("PT_NO_ZSKIP") != nullptr;
      if (&S == &c->newton && gpath && io.f && !no_zskip) {
        if (c->L * Ract > c->zflag_cap) {
          if (c->zflag_d) cudaFree(c->zflag_d);
          c->zflag_d = nullptr;
          CK(cudaMalloc(&c->zflag_d, sizeof(int) * (size_t)c->L * Ract));
          c->zflag_cap = c->L * Ract;
          c->gen++;  // graphs captured with the old buffer are stale
        }
        k_slab_flags<<<dim3(c->L, Ract), 256, 0, c->st>>>(io.f, io.f_stride, c->lay_d, c->wx, Ract, c->zflag_d);
        CK(cudaGetLastError());
        kp.zflag = c->zflag_d;
        if (c->prof) {  // executed-work accounting (profiling runs eagerly): only the tasks that are not skipped
          std::vector<int> fl((size_t)c->L * Ract);
          CK(cudaMemcpyAsync(fl.data(), c->zflag_d, sizeof(int) * fl.size(), cudaMemcpyDeviceToHost, c->st));
          CK(cudaStreamSynchronize(c->st));
          const int gq = T->nc * T->cm;
          long long live = 0, tot = 0;
          for (size_t g = 0; g < S.lgrp.size(); ++g) {
            const int l = S.lgrp[g].first, b = S.lgrp[g].second;
            const int e = g + 1 < S.lgrp.size() ? S.lgrp[g + 1].second : (int)S.ljobs.size();
            const int n = (e - b) * Ract;
            for (int q0 = 0; q0 < n; q0 += gq, ++tot) {
              bool any = false;
              for (int q = q0; q < std::min(n, q0 + gq); ++q) any |= fl[(size_t)l * Ract + q % Ract] != 0;
              live += any;
            }
          }
          const double skipped = tot > 0 ? 1.0 - (double)live / (double)tot : 0.0;
          c->cls_flops[0] -= skipped * T->bytes / 4.0;
          c->cls_bytes[0] -= skipped * T->hbytes;
        }
      }
      CK(k1_launch(kp, T->n, T->nc, c->wmax, c->st));
      c->k1_bytes += T->bytes;
    }
    InnerParams ip = inner_params(c, S, Ract, io);
    ip.rhs_ready = rhs_out;
    c->cls_bytes[1] += S.in_bytes;
    if (c->lu_d) {  // direct inner backend: one dense product per layer solve (nested.py:156-254)
      LaunchScope ls(c, 1);
      const int mmax = 2 * (c->Lc - 1) * c->wmax;
      k_inner_lu<<<dim3((mmax + 7) / 8, J, (Ract + 15) / 16), P0_KQ * 32, 0, c->st>>>(
          S.stage_jobs_d, S.jobs_d, c->lay_d, c->lu_d, c->tables, c->trc, Ract, c->Lc, c->wmax, c->cnt_d);
      CK(cudaGetLastError());
    } else {
      LaunchScope ls(c, 1);
      static const bool no_coop = std::getenv("PT_NO_COOP") != nullptr;
      cudaError_t e = no_coop ? cudaErrorNotSupported : inner_coop_launch(ip, J, c->st);
      if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        e = inner_launch(ip, J, c->st);
      }
      CK(e);
    }
    if (ip.tprof) inner_tprof_dump(S.name);
  }
  if (gpath) {
    c->cls_flops[3] += S.gs_fpr * Ract;
    c->cls_bytes[3] += S.gs_bytes;
    LaunchScope ls(c, 3);
    CK(green_samples_launch(S.jobs_d, J, c->cel_d, c->lay_d, c->gsmp_d, c->trc, c->smp, Ract, c->Lc, c->wx,
                            c->wmax, c->wzcmax, c->num_sms, c->st, fuse_comb ? &tab : nullptr, c->rmap_d));
  } else {
    kp.pass = 1;
    kp.s0 = 0;
    c->cls_flops[0] += T->bytes / 4.0;
    c->cls_bytes[0] += T->hbytes;
    LaunchScope ls(c, 0);
    CK(k1_launch(kp, T->n, T->nc, c->wmax, c->st));
    c->k1_bytes += T->bytes;
  }
  if (tprof_on) {
    long long tt[6];
    cudaStreamSynchronize(c->st);
    cudaMemcpy(tt, tprof_d, sizeof(tt), cudaMemcpyDeviceToHost);
    fprintf(stderr, "K1 tprof nc=%d ntasks=%d: prologue %lld preload %lld bar1 %lld matvec %lld bar2 %lld epi %lld\n",
            T->nc, T->n, tt[0], tt[1], tt[2], tt[3], tt[4], tt[5]);
  }
  if (!c->asm_touch.empty() && S.samples_only && S.no_volume)  // boundary_samples calls (nested.py:356-359)
    for (const OJob& jb : S.jobs) c->touch_extra += c->asm_touch[jb.layer] * Ract;
  if (S.any_sample && !fuse_comb) {
    LaunchScope ls(c, 2);
    k_combine<<<grid_for((long long)J * 4 * Ract * c->wx), 256, 0, c->st>>>(S.jobs_d, J, tab, c->rmap_d, Ract, c->wx,
                                                                              c->smp);
    CK(cudaGetLastError());
  }
  c->layer_solves += (long long)J * Ract;
  return 0;
}

static int lincomb(pt_ctx* c, VecView d, long long doff, VecView x, long long xoff, double a, VecView y,
                   long long yoff, double b, int use_y, long long len, int Ract) {
  if (len <= 0 || Ract == 0) return 0;
  LaunchScope ls(c, 2);
  k_lincomb<<<grid_for(len * Ract), 256, 0, c->st>>>(d, doff, x, xoff, a, y, yoff, b, use_y, len, c->rmap_d, Ract);
  CK(cudaGetLastError());
  return 0;
}

// y = P v  (sie.py:322-329); aux is scratch
static int apply_pre(pt_ctx* c, VecView in, VecView out, VecView aux, int Ract, int gs, const SolveIO& io) {
  const long long wx = c->wx;
  const int nI = c->nI;
  const long long up0 = 2LL * nI * wx;
  int rc = lincomb(c, out, 0, in, 0, -1.0, in, 0, 0.0, 0, 2 * wx, Ract);  // y_down[0] = -v_down[0]
  if (rc) return rc;
  for (int I = 1; I < nI; ++I)
    if ((rc = run_stage(c, c->sdown[I], VecTab{{in, out, aux}}, Ract, io))) return rc;
  VecView sview = in;
  if (gs) {
    if ((rc = run_stage(c, c->refl, VecTab{{out, aux, aux}}, Ract, io))) return rc;
    if ((rc = lincomb(c, aux, up0, in, up0, 1.0, aux, up0, -1.0, 1, up0, Ract))) return rc;  // s = p - refl
    sview = aux;
  }
  if ((rc = lincomb(c, out, up0 + 2LL * (nI - 1) * wx, sview, up0 + 2LL * (nI - 1) * wx, -1.0, sview, 0, 0.0, 0,
                    2 * wx, Ract)))
    return rc;
  for (int I = nI - 2; I >= 0; --I)
    if ((rc = run_stage(c, c->sup[I], VecTab{{sview, out, aux}}, Ract, io))) return rc;
  return 0;
}

static int apply_op(pt_ctx* c, VecView in, VecView out, int Ract, const SolveIO& io) {
  return run_stage(c, c->op, VecTab{{in, out, out}}, Ract, io);
}

static int set_active(pt_ctx* c, const std::vector<int>& a) {
  c->act = a;
  // the pinned staging rotates over PT_RMAP_SLOTS copies: an asynchronous copy still queued behind kernels
  // never sees its source rewritten by a later set_active (a solve synchronises far more often than that)
  int* h = c->hrmap + (size_t)(c->rmap_slot++ % PT_RMAP_SLOTS) * c->capR;
  for (size_t i = 0; i < a.size(); ++i) h[i] = a[i];
  if (!a.empty()) CK(cudaMemcpyAsync(c->rmap_d, h, sizeof(int) * a.size(), cudaMemcpyHostToDevice, c->st));
  return 0;
}

static int grow_outer_basis(pt_ctx* c, int R, int need) {
  if (need <= c->capO) return 0;
  int ncap = std::max(need, 2 * c->capO);
  double2* nv = nullptr;
  CK(cudaMalloc(&nv, sizeof(double2) * (size_t)c->capR * (ncap + 1) * c->nO));
  for (int r = 0; r < R; ++r)
    CK(cudaMemcpyAsync(nv + (size_t)r * (ncap + 1) * c->nO, c->V + (size_t)r * (c->capO + 1) * c->nO,
                       sizeof(double2) * (size_t)(c->capO + 1) * c->nO, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));
  cudaFree(c->V);
  c->V = nv;
  // per-RHS small buffers sized by capO
  cudaFree(c->hout);
  cudaFree(c->ybuf);
  cudaFreeHost(c->hhout);
  cudaFreeHost(c->hy);
  CK(cudaMalloc(&c->hout, sizeof(double2) * (size_t)c->capR * (ncap + 2)));
  CK(cudaMalloc(&c->ybuf, sizeof(double2) * (size_t)c->capR * (ncap + 1)));
  CK(cudaMallocHost(&c->hhout, sizeof(double2) * (size_t)c->capR * (ncap + 2)));
  CK(cudaMallocHost(&c->hy, sizeof(double2) * (size_t)c->capR * (ncap + 1)));
  c->capO = ncap;
  c->gen++;
  return 0;
}

static int check_err(pt_ctx* c, int* code) {
  int e = 0;
  CK(cudaMemcpy(&e, c->err_d, sizeof(int), cudaMemcpyDeviceToHost));
  *code = e;
  return 0;
}

// Run `body` (a launch sequence with no host synchronisation and no host decision on device results) as a
// CUDA graph.  The key names the sequence and every host value it depends on besides c->gen (active count,
// Arnoldi step, io pointers, ...); kernels still read the CURRENT rmap / scalars from device memory.  The
// first sighting runs eagerly, the second captures, instantiates and launches, later ones only launch;
// the host-side counters the body would have advanced are replayed from the capture.  Off while
// profiling (per-launch events), under PT_NO_GRAPH, or after a capture failed.
template <class Body>
static int graphed(pt_ctx* c, std::vector<long long> key, Body&& body) {
  static const bool no_graph = std::getenv("PT_NO_GRAPH") != nullptr || std::getenv("PT_INNER_TPROF") != nullptr ||
                               std::getenv("PT_K1_TPROF") != nullptr;
  if (no_graph || c->prof || c->graphs_off) return body();
  // Executables captured against an older buffer generation can never match again (the key holds the
  // generation), and callers passing fresh device buffers every call add keys: drop the stale ones when the
  // generation moves, and everything when the cache grows past a bound (after the stream drains).
  if (c->graphs_gen != c->gen || c->graphs.size() > 1024) {
    if (!c->graphs.empty()) {
      CK(cudaStreamSynchronize(c->st));
      for (auto& kv : c->graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      c->graphs.clear();
    }
    c->graphs_gen = c->gen;
  }
  key.push_back(c->gen);
  key.push_back((long long)(uintptr_t)c->st);
  pt_ctx::GraphEnt& g = c->graphs[key];
  if (g.exec) {
    CK(cudaGraphLaunch(g.exec, c->st));
    c->layer_solves += g.d_layer_solves;
    c->touch_extra += g.d_touch;
    c->launches += g.d_launches;
    c->k1_launches += g.d_k1_launches;
    c->k1_bytes += g.d_k1_bytes;
    for (int i = 0; i < 5; ++i) {
      c->cls_flops[i] += g.d_cf[i];
      c->cls_bytes[i] += g.d_cb[i];
    }
    return 0;
  }
  if (g.seen++ == 0) return body();
  const long long ls0 = c->layer_solves, la0 = c->launches, k10 = c->k1_launches, tx0 = c->touch_extra;
  const double kb0 = c->k1_bytes;
  double cf0[5], cb0[5];
  for (int i = 0; i < 5; ++i) {
    cf0[i] = c->cls_flops[i];
    cb0[i] = c->cls_bytes[i];
  }
  const long long gen0 = c->gen;
  CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
  const int rc = body();  // records the launches (and advances the host counters by what they will do)
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->st, &graph);
  if (rc == 0 && e == cudaSuccess && c->gen == gen0) e = cudaGraphInstantiate(&g.exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (rc != 0 || e != cudaSuccess || !g.exec) {
    // capture not possible here (e.g. a launch kind the driver cannot capture): eager from now on
    cudaGetLastError();
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    c->graphs_off = true;
    c->layer_solves = ls0;
    c->launches = la0;
    c->k1_launches = k10;
    c->k1_bytes = kb0;
    c->touch_extra = tx0;
    for (int i = 0; i < 5; ++i) {
      c->cls_flops[i] = cf0[i];
      c->cls_bytes[i] = cb0[i];
    }
    return body();
  }
  g.d_layer_solves = c->layer_solves - ls0;
  g.d_touch = c->touch_extra - tx0;
  g.d_launches = c->launches - la0;
  g.d_k1_launches = c->k1_launches - k10;
  g.d_k1_bytes = c->k1_bytes - kb0;
  for (int i = 0; i < 5; ++i) {
    g.d_cf[i] = c->cls_flops[i] - cf0[i];
    g.d_cb[i] = c->cls_bytes[i] - cb0[i];
  }
  CK(cudaGraphLaunch(g.exec, c->st));
  return 0;
}

// ------------------------------------------------------------------ the online solve (sie.py:392-439)

struct RhsState {
  std::vector<cplx> H;  // (m+1) x m column-major, per cycle
  std::vector<cplx> cs, sn, g;
  std::vector<double> hist;
  double beta0 = 0.0;
  int total = 0, k = 0;
  int status = 0;  // 0 running, 1 converged, 2 failed
  double count = -1.0;  // BiCGstab: half steps (reported as the iteration count when >= 0)
};

// Outer BiCGstab (krylov.py:138-201, KrylovConfig.method == "bicgstab") on the device operators for the RHS
// in `run` (beta0 > 0, b = P rhs in Bp, x = 0 in X).  All active RHS advance in lockstep half steps; an RHS
// leaves the active set when it converges.  Vectors live in the outer basis slots: r, r0, p, v, s, t.
// Scalars (vdot, norms) come to the host once per reduction, like the reference's numpy scalars.
static int bicgstab_run(pt_ctx* c, std::vector<RhsState>& rs, std::vector<int>& run, const pt_krylov* cfg, int gs,
                        const SolveIO& io, const long long kio[4]) {
  const int R = c->capR;
  if (grow_outer_basis(c, R, 6)) return PT_CUDA_ERROR;
  const long long nO = c->nO, vs = (long long)(c->capO + 1) * nO;
  VecView vr{c->V + 0 * nO, vs}, vr0{c->V + 1 * nO, vs}, vp{c->V + 2 * nO, vs}, vv{c->V + 3 * nO, vs},
      vsv{c->V + 4 * nO, vs}, vt{c->V + 5 * nO, vs};
  VecView vB{c->Bp, nO}, vX{c->X, nO}, vT{c->T1, nO}, vA{c->AX, nO};
  // coefficients [a | b] and dot outputs [d0 | d1], R complex each, device + pinned host
  double2 *cd = nullptr, *ch = nullptr;
  CK(cudaMalloc(&cd, sizeof(double2) * 4 * R));
  CK(cudaMallocHost(&ch, sizeof(double2) * 4 * R));
  struct Free {
    double2 *d, *h;
    ~Free() {
      cudaFree(d);
      cudaFreeHost(h);
    }
  } fr{cd, ch};
  double2 *ca = cd, *cb = cd + R, *d0 = cd + 2 * R, *d1 = cd + 3 * R;
  auto cx = [](double2 v) { return cplx(v.x, v.y); };
  auto pa = [&](VecView in, VecView out, int Ra, int which) -> int {  // P(A(in)) (krylov.py:151)
    std::vector<long long> key = {5, which, Ra, gs};
    key.insert(key.end(), kio, kio + 4);
    return graphed(c, key, [&]() -> int {
      int r1 = apply_op(c, in, vT, Ra, io);
      if (r1) return r1;
      return apply_pre(c, vT, out, vA, Ra, gs, io);
    });
  };
  auto dots = [&](VecView x0, VecView y0, VecView x1, VecView y1, int two, int Ra) -> int {
    { LaunchScope ls_(c, 2); }
    k_cdot<<<Ra, 256, 0, c->st>>>(x0, y0, nO, c->rmap_d, d0);
    if (two) {
      LaunchScope ls_(c, 2);
      k_cdot<<<Ra, 256, 0, c->st>>>(x1, y1, nO, c->rmap_d, d1);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ch + 2 * R, d0, sizeof(double2) * 2 * R, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return 0;
  };
  auto norms = [&](VecView v, int Ra) -> int {
    { LaunchScope ls_(c, 2); }
    k_norm2<<<Ra, 256, 0, c->st>>>(v, nO, c->rmap_d, c->dscal);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->hdscal, c->dscal, sizeof(double) * R, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return 0;
  };
  auto update = [&](int mode, VecView d, VecView x, VecView y, VecView z, int Ra) -> int {
    CK(cudaMemcpyAsync(cd, ch, sizeof(double2) * 2 * R, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));  // the host rewrites ch for the next update
    LaunchScope ls_(c, 2);
    k_bicg_update<<<grid_for(nO * Ra), 256, 0, c->st>>>(mode, d, x, y, z, ca, cb, nO, c->rmap_d, Ra);
    CK(cudaGetLastError());
    return 0;
  };
  int rc = 0;
  if (run.empty()) return 0;
  if ((rc = set_active(c, run))) return rc;
  int Ra = (int)run.size();
  // r = b, r0 = r (x0 = 0, krylov.py:155-157)
  if ((rc = lincomb(c, vr, 0, vB, 0, 1.0, vB, 0, 0.0, 0, nO, Ra))) return rc;
  if ((rc = lincomb(c, vr0, 0, vB, 0, 1.0, vB, 0, 0.0, 0, nO, Ra))) return rc;
  std::vector<cplx> rho(R, cplx(1, 0)), alpha(R, cplx(1, 0)), omega(R, cplx(1, 0)), beta(R, cplx(0, 0));
  for (int r : run) {
    rs[r].hist.push_back(1.0);  // norm(r) / beta0 with r = b
    rs[r].count = 0.0;
  }
  double count = 0.0;
  const int nit = (int)std::ceil((double)cfg->max_iter);
  for (int it = 0; it < nit && !run.empty(); ++it) {
    if ((rc = set_active(c, run))) return rc;
    Ra = (int)run.size();
    // rho_new = vdot(r0, r) (krylov.py:163)
    if ((rc = dots(vr0, vr, vr0, vr, 0, Ra))) return rc;
    for (int r : run) {
      const cplx rn = cx(ch[2 * R + r]);
      if (std::abs(rn) < 1e-300 * rs[r].beta0 * rs[r].beta0) {
        g_err = "BiCGstab breakdown (rho ~ 0)";
        return PT_BREAKDOWN;
      }
      beta[r] = count > 0 ? (rn / rho[r]) * (alpha[r] / omega[r]) : cplx(0, 0);
      rho[r] = rn;
      ch[r] = make_double2(beta[r].real(), beta[r].imag());
      ch[R + r] = make_double2(omega[r].real(), omega[r].imag());
    }
    // p = r + beta (p - omega v), or p = r on the first step
    if (count > 0) {
      if ((rc = update(1, vp, vr, vv, vv, Ra))) return rc;
    } else if ((rc = lincomb(c, vp, 0, vr, 0, 1.0, vr, 0, 0.0, 0, nO, Ra))) {
      return rc;
    }
    if ((rc = pa(vp, vv, Ra, 0))) return rc;  // v = P A p
    if ((rc = dots(vr0, vv, vr0, vv, 0, Ra))) return rc;
    for (int r : run) {
      const cplx den = cx(ch[2 * R + r]);
      if (std::abs(den) < 1e-300 * rs[r].beta0 * rs[r].beta0) {
        g_err = "BiCGstab breakdown (r0.v ~ 0)";
        return PT_BREAKDOWN;
      }
      alpha[r] = rho[r] / den;
      ch[r] = make_double2(-alpha[r].real(), -alpha[r].imag());
    }
    if ((rc = update(0, vsv, vr, vv, vv, Ra))) return rc;  // s = r - alpha v
    count += 0.5;
    if ((rc = norms(vsv, Ra))) return rc;
    std::vector<int> done, cont;
    for (int r : run) {
      const double res = std::sqrt(c->hdscal[r]) / rs[r].beta0;
      rs[r].hist.push_back(res);
      rs[r].count = count;
      (res <= cfg->ktol ? done : cont).push_back(r);
    }
    if (!done.empty()) {  // x = x + alpha p (krylov.py:180-182)
      if ((rc = set_active(c, done))) return rc;
      for (int r : done) {
        ch[r] = make_double2(alpha[r].real(), alpha[r].imag());
        rs[r].status = 1;
      }
      if ((rc = update(0, vX, vX, vp, vp, (int)done.size()))) return rc;
    }
    run = cont;
    if (run.empty()) break;
    if ((rc = set_active(c, run))) return rc;
    Ra = (int)run.size();
    if ((rc = pa(vsv, vt, Ra, 1))) return rc;  // t = P A s
    if ((rc = dots(vt, vt, vt, vsv, 1, Ra))) return rc;
    for (int r : run) {
      const cplx tt = cx(ch[2 * R + r]), ts = cx(ch[3 * R + r]);
      if (std::abs(tt) == 0.0) {
        g_err = "BiCGstab breakdown (t = 0)";
        return PT_BREAKDOWN;
      }
      omega[r] = ts / tt;
      ch[r] = make_double2(alpha[r].real(), alpha[r].imag());
      ch[R + r] = make_double2(omega[r].real(), omega[r].imag());
    }
    if ((rc = update(2, vX, vX, vp, vsv, Ra))) return rc;  // x = x + alpha p + omega s
    for (int r : run) ch[r] = make_double2(-omega[r].real(), -omega[r].imag());
    if ((rc = update(0, vr, vsv, vt, vt, Ra))) return rc;  // r = s - omega t
    count += 0.5;
    if ((rc = norms(vr, Ra))) return rc;
    cont.clear();
    for (int r : run) {
      const double res = std::sqrt(c->hdscal[r]) / rs[r].beta0;
      rs[r].hist.push_back(res);
      rs[r].count = count;
      if (res <= cfg->ktol)
        rs[r].status = 1;
      else
        cont.push_back(r);
    }
    run = cont;
    if (count >= cfg->max_iter) break;
  }
  for (int r : run) rs[r].status = 2;
  run.clear();
  return 0;
}

static int solve_device(pt_ctx* c, const double2* f, int R, const pt_krylov* cfg, double2* u, pt_stats* stats) {
  if (R <= 0) return PT_BAD_ARGUMENT;
  if (cfg->ktol <= 0 || cfg->max_iter < 1) {
    g_err = "ktol must be positive and max_iter >= 1";
    return PT_BAD_ARGUMENT;
  }
  const long long N = (long long)c->wz * c->wx;
  const int gs = cfg->precond == 0;
  const int max_iter = cfg->max_iter;
  const int cycle = cfg->restart > 0 ? cfg->restart : max_iter;
  if (ensure_scratch(c, R, std::min(max_iter, 16))) return PT_CUDA_ERROR;
  CK(cudaMemsetAsync(c->err_d, 0, sizeof(int), c->st));
  CK(cudaMemsetAsync(c->cnt_d, 0, sizeof(unsigned long long) * 4, c->st));
  CK(cudaMemsetAsync(c->hist_d, 0, sizeof(int) * PT_HIST, c->st));
  c->layer_solves = 0;
  c->touch_extra = 0;
  c->launches = c->k1_launches = 0;
  c->k1_bytes = 0.0;
  for (int i = 0; i < 5; ++i) c->cls_flops[i] = c->cls_bytes[i] = 0.0;
  c->evs.clear();
  c->ev_next = 0;
  static const bool stage_prof = std::getenv("PT_STAGE_PROF") != nullptr;
  if (stage_prof) c->prof = true;
  c->cur_tag = "outer";
  struct EvPair {  // released on every return path
    cudaEvent_t a = nullptr, b = nullptr;
    ~EvPair() {
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } evp;
  CK(cudaEventCreate(&evp.a));
  CK(cudaEventCreate(&evp.b));
  cudaEvent_t e0 = evp.a, e1 = evp.b;
  cudaEventRecord(e0, c->st);

  SolveIO io{f, N, u, N, cfg->inner_ktol, cfg->inner_max_iter};
  const long long kio[4] = {(long long)(uintptr_t)f, (long long)(uintptr_t)u, cfg->inner_max_iter,
                            (long long)(cfg->inner_ktol * 1e15)};
  auto gkey = [&](std::initializer_list<long long> a) {
    std::vector<long long> k(a);
    k.insert(k.end(), kio, kio + 4);
    return k;
  };
  // zero-source detection (sie.py:397-399)
  CK(cudaMemsetAsync(c->dscal, 0, sizeof(double) * 2 * R, c->st));
  { LaunchScope ls_(c, 2); }
  k_vol_norm2<<<dim3(64, R), 256, 0, c->st>>>(f, N, N, c->dscal);
  CK(cudaMemcpyAsync(c->hdscal, c->dscal, sizeof(double) * R, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  std::vector<RhsState> rs(R);
  std::vector<int> live;
  for (int r = 0; r < R; ++r) {
    if (c->hdscal[r] == 0.0) {
      rs[r].status = 1;
      rs[r].hist = {0.0};
      CK(cudaMemsetAsync(u + (size_t)r * N, 0, sizeof(double2) * N, c->st));
    } else {
      live.push_back(r);
    }
  }
  const long long nO = c->nO;
  const long long vstride = (long long)(c->capO + 1) * nO;
  VecView vB{c->Bv, nO}, vBp{c->Bp, nO}, vT{c->T1, nO}, vA{c->AX, nO}, vX{c->X, nO}, vTR{c->TR, nO};
  int rc = 0;
  bool staged = false;  // traces / polarized solution on their way to c->hstage
  // stage buffers index f/u by compact q: the stage kernels read f via rmap-free indexing, so
  // run the volumetric stages with f/u views offset per active list (contiguous when all live).
  std::vector<int> all(R);
  for (int r = 0; r < R; ++r) all[r] = r;

  if (c->nI == 0) {
    // monolayer (sie.py:401-404): reconstruct with empty traces
    if ((rc = set_active(c, all))) return rc;
    if ((rc = run_stage(c, c->recon, VecTab{{vTR, vTR, vTR}}, R, io))) return rc;
    for (int r : live) rs[r].status = 1;
  } else if (!live.empty()) {
    if ((rc = set_active(c, all))) return rc;
    CK(cudaMemsetAsync(c->Bv, 0, sizeof(double2) * (size_t)R * nO, c->st));
    c->tables_f_ok = false;
    // the Newton tables of f alone: RECON's first pass is these plus the pass-0 product of its panels
    const bool keep_tables = c->q0_d && c->Lc > 1 && c->newton.jobs.size() == c->recon.jobs.size();
    rc = graphed(c, gkey({2, R, keep_tables}), [&]() -> int {
      int r2 = run_stage(c, c->newton, VecTab{{vB, vB, vB}}, R, io);
      if (r2) return r2;
      if (keep_tables)
        CK(cudaMemcpyAsync(c->tables_f, c->tables,
                           sizeof(double2) * c->newton.jobs.size() * c->Lc * 4 * (size_t)R * c->wmax,
                           cudaMemcpyDeviceToDevice, c->st));
      return 0;
    });
    if (rc) return rc;
    if (keep_tables) {
      c->tables_f_ok = true;
      c->tables_f_R = R;
    }
    if ((rc = set_active(c, live))) return rc;
    const int Rl = (int)live.size();
    rc = graphed(c, gkey({3, Rl, gs}), [&]() -> int {
      int r3 = apply_pre(c, vB, vBp, vA, Rl, gs, io);
      if (r3) return r3;
      { LaunchScope ls_(c, 2); }
      k_norm2<<<Rl, 256, 0, c->st>>>(vBp, nO, c->rmap_d, c->dscal);
      CK(cudaGetLastError());
      return 0;
    });
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->hdscal, c->dscal, sizeof(double) * R, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemsetAsync(c->X, 0, sizeof(double2) * (size_t)R * nO, c->st));
    CK(cudaStreamSynchronize(c->st));
    int ecode = 0;
    if ((rc = check_err(c, &ecode))) return rc;
    if (ecode) return ecode;
    std::vector<int> run;
    for (int r : live) {
      rs[r].beta0 = std::sqrt(c->hdscal[r]);
      if (rs[r].beta0 == 0.0) {
        rs[r].status = 1;
        rs[r].hist = {0.0};
      } else {
        run.push_back(r);
      }
    }
    int total = 0;
    if (cfg->method == 1) {
      if ((rc = bicgstab_run(c, rs, run, cfg, gs, io, kio))) return rc;
    }
    while (total < max_iter && !run.empty()) {
      if ((rc = set_active(c, run))) return rc;
      int Ra = (int)run.size();
      VecView vV0{c->V, (long long)(c->capO + 1) * nO};
      // r = b - pre(op(x)) on restart, else b (krylov.py:73)
      std::vector<double> beta(R, 0.0);
      if (total > 0) {
        if ((rc = apply_op(c, vX, vT, Ra, io))) return rc;
        if ((rc = apply_pre(c, vT, vTR, vA, Ra, gs, io))) return rc;
        if ((rc = lincomb(c, vV0, 0, vBp, 0, 1.0, vTR, 0, -1.0, 1, nO, Ra))) return rc;
        { LaunchScope ls_(c, 2); }
        k_norm2<<<Ra, 256, 0, c->st>>>(vV0, nO, c->rmap_d, c->dscal);
        CK(cudaMemcpyAsync(c->hdscal, c->dscal, sizeof(double) * R, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        std::vector<int> keep;
        for (int r : run) {
          beta[r] = std::sqrt(c->hdscal[r]);
          if (beta[r] / rs[r].beta0 <= cfg->ktol) {
            rs[r].hist.push_back(beta[r] / rs[r].beta0);
            rs[r].status = 1;
          } else {
            keep.push_back(r);
          }
        }
        run = keep;
        if (run.empty()) break;
        if ((rc = set_active(c, run))) return rc;
        Ra = (int)run.size();
        for (int r : run) c->hdscal[r] = beta[r];
        CK(cudaMemcpyAsync(c->dscal, c->hdscal, sizeof(double) * R, cudaMemcpyHostToDevice, c->st));
        { LaunchScope ls_(c, 2); }
        k_scale_div<<<grid_for(nO * Ra), 256, 0, c->st>>>(vV0, vV0, nO, c->rmap_d, Ra, c->dscal);
      } else {
        for (int r : run) {
          beta[r] = rs[r].beta0;
          c->hdscal[r] = beta[r];
        }
        CK(cudaMemcpyAsync(c->dscal, c->hdscal, sizeof(double) * R, cudaMemcpyHostToDevice, c->st));
        { LaunchScope ls_(c, 2); }
        k_scale_div<<<grid_for(nO * Ra), 256, 0, c->st>>>(vV0, vBp, nO, c->rmap_d, Ra, c->dscal);
      }
      CK(cudaGetLastError());
      const int m = std::min(cycle, max_iter - total);
      for (int r : run) {
        RhsState& s = rs[r];
        s.H.assign((size_t)(m + 1) * m, cplx(0, 0));
        s.cs.assign(m, cplx(0, 0));
        s.sn.assign(m, cplx(0, 0));
        s.g.assign(m + 1, cplx(0, 0));
        s.g[0] = beta[r];
        s.k = 0;
      }
      std::vector<int> cyc = run;  // RHS taking part in this cycle
      std::vector<int> cont = run;
      for (int j = 0; j < m && !cont.empty(); ++j) {
        if ((rc = grow_outer_basis(c, R, j + 1))) return rc;
        const long long vs = (long long)(c->capO + 1) * nO;
        if ((rc = set_active(c, cont))) return rc;
        Ra = (int)cont.size();
        VecView vj{c->V + (size_t)j * nO, vs}, vj1{c->V + (size_t)(j + 1) * nO, vs};
        const int hld = c->capO + 2;
        rc = graphed(c, gkey({1, j, Ra, gs}), [&]() -> int {
          int r1 = apply_op(c, vj, vT, Ra, io);
          if (r1) return r1;
          if ((r1 = apply_pre(c, vT, vj1, vA, Ra, gs, io))) return r1;
          { LaunchScope ls_(c, 2); }
          static const bool arn1 = std::getenv("PT_ARNOLDI_1CTA") != nullptr;
          if (arn1 || 2 * Ra > 2 * c->num_sms)
            k_arnoldi<<<Ra, 512, 0, c->st>>>(c->V, vs, nO, j, c->rmap_d, c->hout, hld);
          else  // two CTAs per RHS
            k_arnoldi2<<<2 * Ra, 512, 0, c->st>>>(c->V, vs, nO, j, c->rmap_d, c->hout, hld);
          CK(cudaGetLastError());
          return 0;
        });
        if (rc) return rc;
        CK(cudaMemcpyAsync(c->hhout, c->hout, sizeof(double2) * (size_t)R * hld, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        int ecode = 0;
        if ((rc = check_err(c, &ecode))) return rc;
        if (ecode) return ecode;
        ++total;
        std::vector<int> nxt;
        for (int r : cont) {
          RhsState& s = rs[r];
          const double2* hc = c->hhout + (size_t)r * hld;
          cplx* col = &s.H[(size_t)j * (m + 1)];
          for (int i = 0; i <= j; ++i) col[i] = cplx(hc[i].x, hc[i].y);
          const double hn = hc[j + 1].x;
          col[j + 1] = hn;
          for (int i = 0; i < j; ++i) {
            const cplx t = s.cs[i] * col[i] + s.sn[i] * col[i + 1];
            col[i + 1] = -std::conj(s.sn[i]) * col[i] + std::conj(s.cs[i]) * col[i + 1];
            col[i] = t;
          }
          const double a = std::abs(col[j]);
          const double d = std::sqrt(a * a + hn * hn);
          if (d == 0.0) {
            g_err = "GMRES breakdown: zero Hessenberg column";
            return PT_BREAKDOWN;
          }
          s.cs[j] = std::conj(col[j]) / d;
          s.sn[j] = hn / d;
          col[j] = s.cs[j] * col[j] + s.sn[j] * hn;
          s.g[j + 1] = -std::conj(s.sn[j]) * s.g[j];
          s.g[j] = s.cs[j] * s.g[j];
          s.k = j + 1;
          s.total = total;
          const double res = std::abs(s.g[j + 1]) / s.beta0;
          s.hist.push_back(res);
          if (hn == 0.0) {
            if (res > cfg->ktol) {
              g_err = "GMRES happy breakdown before convergence";
              return PT_BREAKDOWN;
            }
            continue;  // stops this RHS's cycle
          }
          c->hdscal[r] = hn;
          if (res <= cfg->ktol) continue;
          nxt.push_back(r);
        }
        // normalise V_{j+1} for RHS with hn > 0 (also for the ones that just converged: harmless)
        std::vector<int> norm;
        for (int r : cont)
          if (rs[r].k == j + 1 && c->hdscal[r] > 0.0 && std::abs(rs[r].g[j + 1]) / rs[r].beta0 > cfg->ktol)
            norm.push_back(r);
        if (!norm.empty()) {
          if ((rc = set_active(c, norm))) return rc;
          CK(cudaMemcpyAsync(c->dscal, c->hdscal, sizeof(double) * R, cudaMemcpyHostToDevice, c->st));
          { LaunchScope ls_(c, 2); }
          k_scale_div<<<grid_for(nO * (long long)norm.size()), 256, 0, c->st>>>(vj1, vj1, nO, c->rmap_d,
                                                                                  (int)norm.size(), c->dscal);
          CK(cudaGetLastError());
        }
        cont = nxt;
      }
      // x += V_k y per RHS of this cycle (krylov.py:128-131)
      const int yld = c->capO + 1;
      int kmax = 0;
      for (int r : cyc) {
        RhsState& s = rs[r];
        const int k = s.k;
        kmax = std::max(kmax, k);
        std::vector<cplx> y(k);
        for (int i = k - 1; i >= 0; --i) {
          cplx acc = s.g[i];
          for (int l = i + 1; l < k; ++l) acc -= s.H[(size_t)l * (m + 1) + i] * y[l];
          y[i] = acc / s.H[(size_t)i * (m + 1) + i];
        }
        for (int i = 0; i < yld; ++i) c->hy[(size_t)r * yld + i] = make_double2(0, 0);
        for (int i = 0; i < k; ++i) c->hy[(size_t)r * yld + i] = make_double2(y[i].real(), y[i].imag());
      }
      if ((rc = set_active(c, cyc))) return rc;
      CK(cudaMemcpyAsync(c->ybuf, c->hy, sizeof(double2) * (size_t)R * yld, cudaMemcpyHostToDevice, c->st));
      const long long vs = (long long)(c->capO + 1) * nO;
      { LaunchScope ls_(c, 2); }
      k_accum_x<<<grid_for(nO * (long long)cyc.size()), 256, 0, c->st>>>(vX, c->V, vs, nO, c->ybuf, yld, kmax,
                                                                          c->rmap_d, (int)cyc.size());
      CK(cudaGetLastError());
      std::vector<int> keep;
      for (int r : cyc) {
        if (!rs[r].hist.empty() && rs[r].hist.back() <= cfg->ktol)
          rs[r].status = 1;
        else
          keep.push_back(r);
      }
      run = keep;
    }
    for (int r : run) rs[r].status = 2;  // not converged within max_iter
    // traces = down + up (sie.py:426-427), then reconstruct (sie.py:428)
    if ((rc = set_active(c, all))) return rc;
    const long long half = nO / 2;
    if ((rc = lincomb(c, vTR, 0, vX, 0, 1.0, vX, half, 1.0, 1, half, R))) return rc;
    // the reassembled traces and the polarized solution are final here: they go to pinned staging on a side
    // stream while the reconstruction runs, and reach the caller's arrays before the final synchronisation
    if (stats && (stats->traces || stats->polarized)) {
      const size_t need = (size_t)R * (nO / 2 + nO);
      if (need > c->hstage_cap) {
        if (c->hstage) cudaFreeHost(c->hstage);
        c->hstage = nullptr;
        c->hstage_cap = 0;
        CK(cudaMallocHost(&c->hstage, sizeof(double2) * need));
        c->hstage_cap = need;
      }
      CK(cudaEventRecord(c->ev_tr, c->st));
      CK(cudaStreamWaitEvent(c->side_st, c->ev_tr, 0));
      CK(cudaMemcpy2DAsync(c->hstage, sizeof(double2) * nO / 2, c->TR, sizeof(double2) * nO, sizeof(double2) * nO / 2,
                           R, cudaMemcpyDeviceToHost, c->side_st));
      CK(cudaMemcpyAsync(c->hstage + (size_t)R * nO / 2, c->X, sizeof(double2) * (size_t)R * nO,
                         cudaMemcpyDeviceToHost, c->side_st));
      CK(cudaEventRecord(c->ev_cp, c->side_st));
      staged = true;
    }
    rc = graphed(c, gkey({6, R, c->tables_f_ok, c->tables_f_R}), [&]() -> int {
      return run_stage(c, c->recon, VecTab{{vTR, vTR, vTR}}, R, io);
    });
    if (rc) return rc;
  }
  // residuals (sie.py:441-445)
  if ((rc = set_active(c, all))) return rc;
  CK(cudaMemsetAsync(c->dscal, 0, sizeof(double) * 2 * R, c->st));
  { LaunchScope ls_(c, 2); }
  k_residual<<<dim3(64, R), 256, 0, c->st>>>(u, f, N, c->wz, c->wx, c->tx_d, c->tz_d, c->m_d, c->omega * c->omega,
                                             c->rmap_d, c->dscal, c->hd_d);
  CK(cudaGetLastError());
  cudaEventRecord(e1, c->st);
  CK(cudaMemcpyAsync(c->hdscal, c->dscal, sizeof(double) * 2 * R, cudaMemcpyDeviceToHost, c->st));
  if (staged) {  // host copies from the staging overlap the reconstruction still running on the device
    CK(cudaEventSynchronize(c->ev_cp));
    if (stats->traces)
      std::memcpy(stats->traces, c->hstage, sizeof(double2) * (size_t)R * nO / 2);
    if (stats->polarized)
      std::memcpy(stats->polarized, c->hstage + (size_t)R * nO / 2, sizeof(double2) * (size_t)R * nO);
  } else if (stats && c->nI > 0) {  // nothing solved (monolayer / all sources zero): zero traces
    if (stats->traces) std::memset(stats->traces, 0, sizeof(double2) * (size_t)R * nO / 2);
    if (stats->polarized) std::memset(stats->polarized, 0, sizeof(double2) * (size_t)R * nO);
  }
  CK(cudaStreamSynchronize(c->st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  int ecode = 0;
  if ((rc = check_err(c, &ecode))) return rc;
  if (stats) {
    for (int r = 0; r < R; ++r) {
      const RhsState& s = rs[r];
      if (stats->iterations) stats->iterations[r] = s.count >= 0.0 ? s.count : (double)s.total;
      // the history buffer holds pt_residuals_stride(cfg) entries per RHS: GMRES writes at most max_iter + 1
      // (krylov.py:76-78 appends a cycle-start check), BiCGstab 2 max_iter + 1 (the initial 1.0 and two half
      // steps per iteration, krylov.py:159-199); n_residuals never exceeds what was stored
      const int rstride = pt_residuals_stride(cfg);
      const int nst = (int)std::min(s.hist.size(), (size_t)rstride);
      if (stats->n_residuals) stats->n_residuals[r] = nst;
      if (stats->residuals)
        for (int i = 0; i < nst; ++i) stats->residuals[(size_t)r * rstride + i] = s.hist[i];
      const double ff = c->hdscal[2 * r + 1];
      if (stats->relres) stats->relres[r] = ff > 0 ? std::sqrt(c->hdscal[2 * r]) / std::sqrt(ff) : 0.0;
      if (stats->converged) stats->converged[r] = s.status == 1;
    }

    unsigned long long cnt[4] = {0, 0, 0, 0};
    CK(cudaMemcpy(cnt, c->cnt_d, sizeof(cnt), cudaMemcpyDeviceToHost));
    if (stats->layer_solves) stats->layer_solves[0] = c->layer_solves;
    if (stats->inner_iters) stats->inner_iters[0] = (long long)cnt[0];
    if (stats->touches) stats->touches[0] = (long long)cnt[1] + c->touch_extra;
    if (stats->inner_hist && stats->inner_hist_len > 0) {
      int hh[PT_HIST];
      CK(cudaMemcpy(hh, c->hist_d, sizeof(hh), cudaMemcpyDeviceToHost));
      for (int i = 0; i < stats->inner_hist_len; ++i) stats->inner_hist[i] = i < PT_HIST ? hh[i] : 0;
    }
    if (stats->timing_ms) stats->timing_ms[0] = ms;
    if (stats->kernel_ms) {
      double acc[5] = {0, 0, 0, 0, 0};
      for (const auto& e : c->evs) {
        float t = 0.f;
        cudaEventElapsedTime(&t, e.a, e.b);
        acc[e.cls] += t;
      }
      stats->kernel_ms[0] = acc[0];
      stats->kernel_ms[1] = acc[1];
      stats->kernel_ms[2] = c->prof ? std::max(0.0, (double)ms - acc[0] - acc[1]) : 0.0;
    }
    if (stage_prof) {  // per (stage, kernel class) device time, launch count
      std::map<std::string, std::pair<double, int>> agg;
      static const char* cls_name[5] = {"k1", "inner", "glue", "green", "pass0"};
      for (const auto& e : c->evs) {
        float t = 0.f;
        cudaEventElapsedTime(&t, e.a, e.b);
        auto& v = agg[std::string(e.tag) + "/" + cls_name[e.cls]];
        v.first += t;
        v.second += 1;
      }
      double ksum = 0.0;
      for (const auto& kv : agg) ksum += kv.second.first;
      fprintf(stderr, "stage profile (total %.3f ms, launches %.3f ms, gaps %.3f ms):\n", ms, ksum, ms - ksum);
      for (const auto& kv : agg)
        fprintf(stderr, "  %-16s %8.3f ms  %5d launches  %8.1f us/launch\n", kv.first.c_str(), kv.second.first,
                kv.second.second, 1e3 * kv.second.first / kv.second.second);
    }
    if (stats->k1_bytes) stats->k1_bytes[0] = c->k1_bytes;
    if (stats->class_ms) {
      double acc5[5] = {0, 0, 0, 0, 0};
      for (const auto& e : c->evs) {
        float t = 0.f;
        cudaEventElapsedTime(&t, e.a, e.b);
        acc5[e.cls] += t;
      }
      for (int i = 0; i < 5; ++i) stats->class_ms[i] = acc5[i];
    }
    if (stats->dense_flops) {
      // dense inner products: pre(rhs) once and pre(op(.)) once per inner iteration, per instance
      double f = 0.0;
      if (c->dense_d) {
        const double n = 4.0 * (c->Lc - 1) * c->wmax;  // n from the widest layer (exact when all are equal)
        f = 8.0 * n * n * (double)(cnt[0] + (long long)c->layer_solves);
      }
      stats->dense_flops[0] = f;
    }
    if (stats->launches) stats->launches[0] = c->launches;
    if (stats->k1_launches) stats->k1_launches[0] = c->k1_launches;
    if (stats->class_flops) {
      for (int i = 0; i < 5; ++i) stats->class_flops[i] = c->cls_flops[i];
      // inner GMRES: dense products (8 n^2 per instance and product) or the Green-block touches x 8
      stats->class_flops[1] = c->dense_d ? (stats->dense_flops ? stats->dense_flops[0] : 0.0)
                                         : 8.0 * (double)((long long)cnt[1] + c->touch_extra);
      if (c->dense_d && !stats->dense_flops) {
        const double n = 4.0 * (c->Lc - 1) * c->wmax;
        stats->class_flops[1] = 8.0 * n * n * (double)(cnt[0] + (long long)c->layer_solves);
      }
    }
    if (stats->class_bytes)
      for (int i = 0; i < 5; ++i) stats->class_bytes[i] = c->cls_bytes[i];
  }
  if (ecode) return ecode;
  for (int r = 0; r < R; ++r)
    if (rs[r].status == 2) {
      g_err = "outer GMRES did not reach ktol within max_iter";
      return PT_NOT_CONVERGED;
    }
  return PT_OK;
}

// ------------------------------------------------------------------ C ABI

extern "C" {

const char* pt_last_error(void) { return g_err.c_str(); }
const char* pt_version(void) { return "pt_b200 0.2 (sm_100a)"; }

int pt_residuals_stride(const pt_krylov* cfg) {
  if (!cfg || cfg->max_iter < 1) return 0;
  return cfg->method == 1 ? 2 * cfg->max_iter + 1 : cfg->max_iter + 1;
}

static int create_impl(pt_ctx* c, const pt_problem* pb, int device, pt_ctx** out);

// Every failure after the context exists releases it (streams, events, device buffers) through
// pt_destroy, which tolerates the members that were never created.
int pt_create(const pt_problem* pb, int device, pt_ctx** out) {
  if (!pb || !out) return PT_BAD_ARGUMENT;
  *out = nullptr;
  if (pb->L < 1 || pb->Lc < 1 || pb->Lc > PT_MAX_LC || pb->nx < 1 || pb->nz < 1) {
    g_err = "bad problem geometry";
    return PT_BAD_ARGUMENT;
  }
  CK(cudaSetDevice(device));
  pt_ctx* c = new pt_ctx();
  const int rc = create_impl(c, pb, device, out);
  if (rc != PT_OK) {
    const std::string err = g_err;
    *out = nullptr;
    pt_destroy(c);
    g_err = err;
  }
  return rc;
}

static int create_impl(pt_ctx* c, const pt_problem* pb, int device, pt_ctx** out) {
  c->dev = device;
  CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  c->own_st = c->st;
  CK(cudaStreamCreateWithFlags(&c->side_st, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_tr, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_cp, cudaEventDisableTiming));
  c->nx = pb->nx;
  c->nz = pb->nz;
  c->npml = pb->npml;
  c->L = pb->L;
  c->Lc = pb->Lc;
  c->h = pb->h;
  c->omega = pb->omega;
  c->wx = pb->nx + 2 * pb->npml;
  c->wz = pb->nz + 2 * pb->npml;
  c->nI = pb->L - 1;
  if (const char* e = std::getenv("PT_INNER_CAP")) c->inner_cap = std::max(2, atoi(e));
  if (const char* e = std::getenv("PT_COOP_SMS")) c->coop_sms = std::max(0, atoi(e));
  const int npml = c->npml;
  // layers
  int off = 0;
  c->wmax = 0;
  for (int l = 0; l < c->L; ++l) {
    LayerInfo li;
    std::memset(&li, 0, sizeof(li));
    li.n = pb->layer_extents[l];
    li.off = off;
    li.w = li.n + 2 * npml;
    li.lo = l == 0 ? 0 : npml;
    li.hi = l == c->L - 1 ? li.w : npml + li.n;
    li.has_top = l >= 1;
    li.has_bot = l <= c->L - 2;
    const int rowv[4] = {npml, npml - 1, li.n + npml, li.n + npml - 1};  // row(1), row(0), row(n+1), row(n)
    for (int s = 0; s < 4; ++s) {
      li.prow[s] = rowv[s];
      li.coef[s] = make_double2(pb->layer_coefs[(l * 4 + s) * 2], pb->layer_coefs[(l * 4 + s) * 2 + 1]);
    }
    li.dense_off = -1;
    li.lu_off = -1;
    if (li.w > 128) {
      g_err = "layer width n_l + 2 npml exceeds 128 (K1 holds <= 4 rows per lane)";
      return PT_BAD_ARGUMENT;
    }
    c->wmax = std::max(c->wmax, li.w);
    c->lay.push_back(li);
    off += li.n;
  }
  if (off != c->nz) {
    g_err = "layer extents do not sum to nz";
    return PT_BAD_ARGUMENT;
  }
  // scan form of the inner GS sweeps (build_inner): product blocks T^(2), T^(4), ... of the cells' transfer
  // matrices follow the 16 Green blocks of every cell (rows 4 + 2 (level - 1) + s, slots = [down k0, k1, up k0, k1]).
  // Item-program layers only (no dense / direct inner operators); PT_NO_SCAN keeps the sequential sweeps.
  c->scan_levels = 0;
  if (pb->green && !pb->inner_dense && !pb->inner_lu && c->Lc >= 4 && !std::getenv("PT_NO_SCAN")) {
    int nlev = 0;
    while ((1 << nlev) < c->Lc - 1) ++nlev;
    c->scan_levels = nlev - 1;
  }
  // cells
  long long soff = 0, goff = 0, zoff = 0, gsoff = 0, q0off = 0;
  c->wzcmax = 0;
  std::vector<int> coffs(c->Lc);
  {
    int o = 0, sum = 0;
    for (int cc = 0; cc < c->Lc; ++cc) {
      coffs[cc] = o;
      o += pb->cell_extents[cc];
      sum += pb->cell_extents[cc];
    }
    if (sum != c->nx) {
      g_err = "cell extents do not sum to nx";
      return PT_BAD_ARGUMENT;
    }
  }
  for (int l = 0; l < c->L; ++l)
    for (int cc = 0; cc < c->Lc; ++cc) {
      CellInfo ci;
      std::memset(&ci, 0, sizeof(ci));
      ci.layer = l;
      ci.cell = cc;
      ci.w = c->lay[l].w;
      ci.nxc = pb->cell_extents[cc];
      ci.wzc = ci.nxc + 2 * npml;
      ci.off = coffs[cc];
      ci.lo = cc == 0 ? 0 : npml;
      ci.hi = cc == c->Lc - 1 ? ci.wzc : npml + ci.nxc;
      ci.has_top = cc >= 1;
      ci.has_bot = cc <= c->Lc - 2;
      const int n = ci.nxc;
      const int krow[4] = {npml, npml - 1, n + npml, n + npml - 1};
      const int srow[4] = {npml - 1, npml, n + npml - 1, n + npml};
      const int id = l * c->Lc + cc;
      for (int s = 0; s < 4; ++s) {
        ci.krow[s] = krow[s];
        ci.srow[s] = srow[s];
        ci.coef[s] = make_double2(pb->cell_coefs[(id * 4 + s) * 2], pb->cell_coefs[(id * 4 + s) * 2 + 1]);
      }
      ci.sinv_off = soff;
      ci.green_off = goff;
      ci.lz_off = zoff;
      ci.gsmp_off = pb->gsmp ? gsoff : -1;
      gsoff += 16LL * ci.wzc * ci.w;
      {
        const int nk = ci.hi - ci.lo, nk4 = (nk + 3) & ~3;
        const long long mp = q0_rows(ci.w, nk);  // device row layout
        ci.q0_off = pb->q0 ? q0off : -1;
        q0off += mp * 4 * nk4;
      }
      soff += (long long)ci.wzc * ci.w * ((ci.w + 3) & ~3);  // blocks padded to a multiple of 4 columns
      goff += (16LL + 8LL * c->scan_levels) * ((ci.w + 7) / 8) * 8 * ci.w;  // tile-major, rows padded to 8
      zoff += ci.wzc;
      c->wzcmax = std::max(c->wzcmax, ci.wzc);
      c->cel.push_back(ci);
    }
  CK(cudaMalloc(&c->sinv_d, sizeof(double2) * (size_t)soff));
  CK(cudaMalloc(&c->green_d, sizeof(double2) * (size_t)goff));
  if (pb->gsmp) CK(cudaMalloc(&c->gsmp_d, sizeof(double2) * (size_t)gsoff));
  if (pb->q0) CK(cudaMalloc(&c->q0_d, sizeof(double2) * (size_t)q0off));
  CK(cudaMalloc(&c->lz_d, sizeof(double2) * (size_t)zoff));
  CK(cudaMalloc(&c->uz_d, sizeof(double2) * (size_t)zoff));
  for (const CellInfo& ci : c->cel) {
    const int id = ci.layer * c->Lc + ci.cell;
    {
      // column-major blocks, zero-padded from w to w4 = roundup(w, 4) columns (DMMA k-steps of 4)
      const int w4 = (ci.w + 3) & ~3;
      CK(cudaMemset(c->sinv_d + ci.sinv_off, 0, sizeof(double2) * (size_t)ci.wzc * ci.w * w4));
      CK(cudaMemcpy2D(c->sinv_d + ci.sinv_off, sizeof(double2) * (size_t)ci.w * w4, pb->sinv[id],
                      sizeof(double2) * (size_t)ci.w * ci.w, sizeof(double2) * (size_t)ci.w * ci.w, ci.wzc,
                      cudaMemcpyDefault));
    }
    if (!pb->green) {  // factor-only context (the offline stage's own cell solves): no interface operators yet
      CK(cudaMemset(c->green_d + ci.green_off, 0, sizeof(double2) * 16 * (size_t)((ci.w + 7) / 8) * 8 * ci.w));
    } else {
      double2* tmp = nullptr;
      CK(cudaMalloc(&tmp, sizeof(double2) * 16 * (size_t)ci.w * ci.w));
      CK(cudaMemcpy(tmp, pb->green[id], sizeof(double2) * 16 * (size_t)ci.w * ci.w, cudaMemcpyDefault));
      k_green_tiles<<<256, 256>>>(tmp, c->green_d + ci.green_off, ci.w, 16);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      cudaFree(tmp);
    }
    if (pb->gsmp)
      CK(cudaMemcpy(c->gsmp_d + ci.gsmp_off, pb->gsmp[id], sizeof(double2) * 16 * (size_t)ci.wzc * ci.w,
                    cudaMemcpyDefault));
    if (pb->q0) {
      const int nk = ci.hi - ci.lo, nk4 = (nk + 3) & ~3;
      const long long mp = (4LL * ci.w + 4LL * nk + 7) / 8 * 8;  // rows of the ABI array
      double2* tmp = nullptr;
      CK(cudaMalloc(&tmp, sizeof(double2) * (size_t)(mp * 4 * nk4)));
      CK(cudaMemcpy(tmp, pb->q0[id], sizeof(double2) * (size_t)(mp * 4 * nk4), cudaMemcpyDefault));
      k_q0_rows<<<512, 256>>>(tmp, c->q0_d + ci.q0_off, ci.w, nk, 4 * nk4);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      cudaFree(tmp);
    }
    CK(cudaMemcpy(c->lz_d + ci.lz_off, pb->lz[id], sizeof(double2) * ci.wzc, cudaMemcpyDefault));
    CK(cudaMemcpy(c->uz_d + ci.lz_off, pb->uz[id], sizeof(double2) * ci.wzc, cudaMemcpyDefault));
  }
  if (c->scan_levels > 0) {
    const int nI = c->Lc - 1;
    for (int l = 0; l < c->L; ++l) {
      const int w = c->lay[l].w;
      const size_t W = (size_t)w * w, W4 = 4 * W;
      // level matrices [dir][I][s][k][w*w], column-major blocks: dir 0 = T_I (cell I: rows n, n+1; slots v0, v1),
      // dir 1 = U_I (cell I + 1: rows 0, 1; slots vn, vnp)
      double2 *cur = nullptr, *nxt = nullptr, *tmp8 = nullptr;
      CK(cudaMalloc(&cur, sizeof(double2) * 2 * nI * W4));
      CK(cudaMalloc(&nxt, sizeof(double2) * 2 * nI * W4));
      CK(cudaMalloc(&tmp8, sizeof(double2) * 8 * W));
      CK(cudaMemset(cur, 0, sizeof(double2) * 2 * nI * W4));
      for (int cc = 1; cc <= c->Lc - 2; ++cc) {
        const double2* g = reinterpret_cast<const double2*>(pb->green[l * c->Lc + cc]);  // [4 rows][4 slots][w*w]
        for (int sb = 0; sb < 2; ++sb) {
          CK(cudaMemcpy(cur + (size_t)cc * W4 + (size_t)sb * 2 * W, g + (size_t)((2 + sb) * 4 + 0) * W,
                        sizeof(double2) * 2 * W, cudaMemcpyDefault));
          CK(cudaMemcpy(cur + (size_t)(nI + cc - 1) * W4 + (size_t)sb * 2 * W, g + (size_t)(sb * 4 + 2) * W,
                        sizeof(double2) * 2 * W, cudaMemcpyDefault));
        }
      }
      const dim3 mg((w + 15) / 16, (w + 15) / 16, 4), mb(16, 16);
      for (int lv = 1; lv <= c->scan_levels; ++lv) {
        const int st = 1 << (lv - 1);  // stride of the factors; the products have stride 2 st
        CK(cudaMemset(nxt, 0, sizeof(double2) * 2 * nI * W4));
        for (int I = 2 * st; I <= nI - 1; ++I)  // T^(2st)_I = T^(st)_I T^(st)_{I - st}
          k_block2_mm<<<mg, mb>>>(cur + (size_t)I * W4, cur + (size_t)(I - st) * W4, nxt + (size_t)I * W4, w);
        for (int I = 0; I <= nI - 1 - 2 * st; ++I)  // U^(2st)_I = U^(st)_I U^(st)_{I + st}
          k_block2_mm<<<mg, mb>>>(cur + (size_t)(nI + I) * W4, cur + (size_t)(nI + I + st) * W4,
                                  nxt + (size_t)(nI + I) * W4, w);
        CK(cudaGetLastError());
        for (int cc = 0; cc < c->Lc; ++cc) {
          const CellInfo& ci = c->cel[l * c->Lc + cc];
          CK(cudaMemsetAsync(tmp8, 0, sizeof(double2) * 8 * W));
          for (int sb = 0; sb < 2; ++sb) {
            if (cc >= 2 * st && cc <= nI - 1)
              CK(cudaMemcpyAsync(tmp8 + (size_t)(sb * 4 + 0) * W, nxt + (size_t)cc * W4 + (size_t)sb * 2 * W,
                                 sizeof(double2) * 2 * W, cudaMemcpyDeviceToDevice));
            if (cc - 1 >= 0 && cc - 1 <= nI - 1 - 2 * st)
              CK(cudaMemcpyAsync(tmp8 + (size_t)(sb * 4 + 2) * W, nxt + (size_t)(nI + cc - 1) * W4 + (size_t)sb * 2 * W,
                                 sizeof(double2) * 2 * W, cudaMemcpyDeviceToDevice));
          }
          const size_t blk = (size_t)((ci.w + 7) / 8) * 8 * ci.w;  // one tile-major block
          k_green_tiles<<<256, 256>>>(tmp8, c->green_d + ci.green_off + (16 + 8 * (size_t)(lv - 1)) * blk, ci.w, 8);
          CK(cudaGetLastError());
        }
        std::swap(cur, nxt);
      }
      CK(cudaDeviceSynchronize());
      cudaFree(cur);
      cudaFree(nxt);
      cudaFree(tmp8);
    }
  }
  // dense inner operators (optional): [L] x [2][n][n], n = 4 nI w
  if (pb->inner_dense && c->Lc > 1) {
    // stored DMMA-fragment tile-major (k_dense_tiles), rows padded to whole 8-row tiles
    // per layer: [pre | pre o op] and, with the s-step operators, the stack [pre; E pre; E^2 pre] (row tiles of
    // the three stacked in every k chunk, so one streaming pass serves all three)
    const int cnt = pb->inner_dense_count >= 4 ? 4 : 2;
    c->dense_cnt = cnt;
    long long doff = 0;
    for (auto& li : c->lay) {
      const long long n = 4LL * (c->Lc - 1) * li.w;
      li.dense_off = doff;
      doff += (cnt == 4 ? 5 : 2) * dense_matrix_elems(n);
    }
    CK(cudaMalloc(&c->dense_d, sizeof(double2) * (size_t)doff));
    double2* tmp = nullptr;
    const long long nmx = 4LL * (c->Lc - 1) * c->wmax;
    CK(cudaMalloc(&tmp, sizeof(double2) * (size_t)(cnt * nmx * nmx)));
    for (int l = 0; l < c->L; ++l) {
      const long long n = 4LL * (c->Lc - 1) * c->lay[l].w, me = dense_matrix_elems(n);
      CK(cudaMemcpy(tmp, pb->inner_dense[l], sizeof(double2) * (size_t)(cnt * n * n), cudaMemcpyDefault));
      for (int m = 0; m < 2; ++m) {
        k_dense_tiles<<<512, 256>>>(tmp + (size_t)m * n * n, c->dense_d + c->lay[l].dense_off + (size_t)m * me,
                                    (int)n, DA_KC);
        CK(cudaGetLastError());
      }
      if (cnt == 4) {
        k_dense_tiles_stack3<<<512, 256>>>(tmp, tmp + (size_t)2 * n * n, tmp + (size_t)3 * n * n,
                                           c->dense_d + c->lay[l].dense_off + (size_t)2 * me, (int)n, DA_KC);
        CK(cudaGetLastError());
      }
      CK(cudaDeviceSynchronize());
    }
    cudaFree(tmp);
  }
  // direct inner backend (optional): [L] x [m][m], m = 2 nI w, row-major
  if (pb->inner_lu && c->Lc > 1) {
    long long off = 0;
    for (auto& li : c->lay) {
      const long long m = 2LL * (c->Lc - 1) * li.w;
      li.lu_off = off;
      off += m * m;
    }
    CK(cudaMalloc(&c->lu_d, sizeof(double2) * (size_t)off));
    for (int l = 0; l < c->L; ++l) {
      const long long m = 2LL * (c->Lc - 1) * c->lay[l].w;
      CK(cudaMemcpy(c->lu_d + c->lay[l].lu_off, pb->inner_lu[l], sizeof(double2) * (size_t)(m * m), cudaMemcpyDefault));
    }
  }
  if (upload(&c->lay_d, c->lay.data(), c->lay.size())) return PT_CUDA_ERROR;
  if (upload(&c->cel_d, c->cel.data(), c->cel.size())) return PT_CUDA_ERROR;
  if (upload(&c->tx_d, reinterpret_cast<const double2*>(pb->tx), 3 * (size_t)c->wx)) return PT_CUDA_ERROR;
  if (upload(&c->tz_d, reinterpret_cast<const double2*>(pb->tz), 3 * (size_t)c->wz)) return PT_CUDA_ERROR;
  if (upload(&c->m_d, pb->m, (size_t)c->wz * c->wx)) return PT_CUDA_ERROR;
  if (pb->hdiag && upload(&c->hd_d, reinterpret_cast<const double2*>(pb->hdiag), (size_t)c->wz * c->wx))
    return PT_CUDA_ERROR;
  CK(cudaMalloc(&c->err_d, sizeof(int)));
  CK(cudaMalloc(&c->cnt_d, sizeof(unsigned long long) * 4));
  CK(cudaMalloc(&c->hist_d, sizeof(int) * PT_HIST));
  // K1 shared-memory ring: 8 slots (a multiple of every multicast group size), as large as fit
  {
    int maxsm = 0;
    CK(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    c->ns = 8;
    const long long fixed = (long long)k1_smem_bytes(c->wmax, 8, 0, c->ns);
    long long slot = ((long long)maxsm - fixed) / c->ns;
    slot = std::min(slot, 32768LL) / 16 * 16;
    if (slot < 16LL * c->wmax) {
      g_err = "not enough shared memory for the K1 ring";
      return PT_BAD_ARGUMENT;
    }
    c->slot_bytes = (int)slot;
  }
  for (const CellInfo& ci : c->cel)
    if (ci.wzc < 3) {
      g_err = "cells need nx_c + 2 npml >= 3 block rows";
      return PT_BAD_ARGUMENT;
    }
  if (pb->assembled_boundary && c->Lc > 1) {  // nested.py:447-484: M_f, direct and M_u matvecs per call
    c->asm_touch.assign(c->L, 0);
    for (const CellInfo& ci : c->cel) {
      const long long s_ = ci.hi - ci.lo, w = ci.w, nsl = 2 * (ci.has_top + ci.has_bot);
      c->asm_touch[ci.layer] += 16 * w * s_ + 16 * s_ * s_ + 4 * nsl * s_ * w;
    }
  }
  int rc = build_inner(c);
  if (!rc) rc = build_outer(c);
  if (rc) return rc;
  // standalone layer-solve stage (one job per layer, full slab in/out) built on demand
  *out = c;
  return PT_OK;
}

int pt_set_stream(pt_ctx* c, void* stream) {
  if (!c) return PT_BAD_ARGUMENT;
  c->st = stream ? static_cast<cudaStream_t>(stream) : c->own_st;
  return PT_OK;
}

int pt_set_profiling(pt_ctx* c, int enable) {
  if (!c) return PT_BAD_ARGUMENT;
  c->prof = enable != 0;
  return PT_OK;
}

int pt_destroy(pt_ctx* c) {
  if (!c) return PT_OK;
  cudaSetDevice(c->dev);
  cudaDeviceSynchronize();
  // the process-level allocations are released with the context
  for (cudaEvent_t e : c->evpool) cudaEventDestroy(e);
  for (void* p : {(void*)c->lay_d, (void*)c->cel_d, (void*)c->sinv_d, (void*)c->green_d, (void*)c->gsmp_d, (void*)c->q0_d, (void*)c->dense_d, (void*)c->lu_d, (void*)c->lz_d,
                  (void*)c->uz_d, (void*)c->tx_d, (void*)c->tz_d, (void*)c->m_d, (void*)c->hd_d, (void*)c->items_d, (void*)c->items_px_d, (void*)c->pre_ph_px_d, (void*)c->zflag_d,
                  (void*)c->op_ph_d, (void*)c->pre_ph_d, (void*)c->V, (void*)c->Bv, (void*)c->Bp, (void*)c->T1,
                  (void*)c->AX, (void*)c->X, (void*)c->TR, (void*)c->P, (void*)c->smp, (void*)c->tables, (void*)c->tables_f,
                  (void*)c->trc, (void*)c->Z, (void*)c->iscr, (void*)c->hess, (void*)c->iters, (void*)c->istate,
                  (void*)c->ibeta0, (void*)c->err_d,
                  (void*)c->cnt_d, (void*)c->hist_d, (void*)c->rmap_d, (void*)c->dscal, (void*)c->hout,
                  (void*)c->ybuf, (void*)c->io_f, (void*)c->io_u, (void*)c->ipart})
    if (p) cudaFree(p);
  for (void* p : {(void*)c->hrmap, (void*)c->hhout, (void*)c->hdscal, (void*)c->hy})
    if (p) cudaFreeHost(p);
  std::vector<Stage*> stages = {&c->newton, &c->op, &c->refl, &c->recon};
  for (auto& st : c->sdown) stages.push_back(&st);
  for (auto& st : c->sup) stages.push_back(&st);
  for (Stage* st : stages) {
    for (auto& kv : st->tasks) cudaFree(kv.second.d);
    if (st->jobs_d) cudaFree(st->jobs_d);
    if (st->stage_jobs_d) cudaFree(st->stage_jobs_d);
    if (st->ljobs_d) cudaFree(st->ljobs_d);
    if (st->grp_d) cudaFree(st->grp_d);
  }
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  if (c->hstage) cudaFreeHost(c->hstage);
  if (c->ev_tr) cudaEventDestroy(c->ev_tr);
  if (c->ev_cp) cudaEventDestroy(c->ev_cp);
  if (c->side_st) cudaStreamDestroy(c->side_st);
  for (cudaEvent_t e : {c->ev_h2d[0], c->ev_h2d[1], c->ev_done})
    if (e) cudaEventDestroy(e);
  if (c->io_st) cudaStreamDestroy(c->io_st);
  if (c->own_st) cudaStreamDestroy(c->own_st);
  delete c;
  return PT_OK;
}

static int solve_batch(pt_ctx* c, const double* f, int nrhs, const pt_krylov* cfg, double* u, pt_stats* stats) {
  int rc;
  const int need = std::max(2, cfg->inner_max_iter + 1);  // basis vectors of an inner solve at max_iter
  while (true) {
    rc = solve_device(c, reinterpret_cast<const double2*>(f), nrhs, cfg, reinterpret_cast<double2*>(u), stats);
    if (rc != PT_CAPACITY) break;
    if (c->inner_cap >= need) {  // cannot happen: an inner solve stops at inner_max_iter (InnerSolveError)
      g_err = "inner GMRES did not converge within inner_max_iter";
      return PT_INNER_NOT_CONVERGED;
    }
    // an inner Krylov basis outgrew its capacity: grow it (up to inner_max_iter + 1) and redo the solve
    c->inner_cap = std::min(2 * c->inner_cap, need);
    c->capR = 0;
    c->capO = 0;
  }
  return rc;
}

// RHS per lockstep batch: every stage's inner GMRES runs as ONE cooperative launch over its (job, group of
// 8 RHS) units, which holds at most inner_coop_max_units() units (the widest stage has max(2L-2, L) jobs)
static int batch_rhs(const pt_ctx* c) {
  const int maxj = std::max(std::max((int)c->op.jobs.size(), (int)c->newton.jobs.size()),
                            std::max((int)c->recon.jobs.size(), (int)c->refl.jobs.size()));
  if (c->Lc < 2 || maxj == 0) return 1 << 30;
  // item programs (no dense inner operators): every stage runs the all-RHS item kernel (inner_items.cu, up to
  // 256 RHS per job).  The sweep stages are latency-bound, so a batch takes as many RHS as the kernel holds and
  // the memory allows: 64 at least, then 128 / 192 / 256 while the per-RHS scratch (inner Krylov bases of the
  // widest stage, stage panels and tables, staged wavefields) stays below 40 % of the free device memory seen at
  // the first solve (PT_BATCH_RHS overrides).
  if (!c->dense_d && !c->lu_d && maxj <= 64 && !std::getenv("PT_ITEMS_V1")) {
    if (c->batch_cap <= 0) {
      int b = 64;
      if (const char* e = std::getenv("PT_BATCH_RHS")) {
        b = std::max(8, std::min(256, atoi(e) / 8 * 8));
      } else {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
          const double nmax = 4.0 * (c->Lc - 1) * c->wmax;
          // inner Krylov bases sized for twice the default capacity (a capacity retry doubles them)
          const double per = 1.25 * maxj * (std::max(c->inner_cap, 24) + 5) * nmax * 16.0 +
                             2.0 * 16.0 * c->wz * (double)c->wx;
          while (b + 64 <= 256 && per * (b + 64) <= 0.4 * (double)free_b) b += 64;
        }
      }
      const_cast<pt_ctx*>(c)->batch_cap = b;
    }
    return c->batch_cap;
  }
  return 8 * std::max(1, inner_coop_max_units() / maxj);
}

// Host staging of a multi-batch solve (pt_solve): fh / uh are the caller's host arrays, f / u the device staging
// buffers.  Batch b's sources are copied on io_st while batch b - 1 solves, its wavefields while batch b + 1 solves.
struct HostIO {
  const double* fh;
  double* uh;
};

static int solve_batches(pt_ctx* c, const double* f, int nrhs, const pt_krylov* cfg, double* u, pt_stats* stats,
                         const HostIO* hio);

int pt_solve_device(pt_ctx* c, const double* f, int nrhs, const pt_krylov* cfg, double* u, pt_stats* stats) {
  if (!c || !f || !u || !cfg) return PT_BAD_ARGUMENT;
  CK(cudaSetDevice(c->dev));
  return solve_batches(c, f, nrhs, cfg, u, stats, nullptr);
}

static int solve_batches(pt_ctx* c, const double* f, int nrhs, const pt_krylov* cfg, double* u, pt_stats* stats,
                         const HostIO* hio) {
  const int B = batch_rhs(c);
  if (nrhs <= B && !hio) return solve_batch(c, f, nrhs, cfg, u, stats);
  // large source sets: consecutive lockstep batches; per-RHS outputs land at their offsets, totals add up
  const long long N = 2LL * c->wz * c->wx;  // doubles per wavefield
  const long long nO = 4LL * c->nI * c->wx;
  pt_stats acc;
  std::memset(&acc, 0, sizeof(acc));
  long long ls = 0, ii = 0, to = 0, la = 0, k1l = 0;
  double tms = 0, kms[3] = {0, 0, 0}, k1b = 0, cms[5] = {0, 0, 0, 0, 0}, dfl = 0;
  double cf[5] = {0, 0, 0, 0, 0}, cb[5] = {0, 0, 0, 0, 0};
  std::vector<int> hist(stats && stats->inner_hist_len > 0 ? stats->inner_hist_len : 0, 0);
  int worst = PT_OK;
  if (hio) {
    if (!c->io_st) {
      CK(cudaStreamCreateWithFlags(&c->io_st, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
    }
    const int n0 = std::min(B, nrhs);
    CK(cudaMemcpyAsync(const_cast<double*>(f), hio->fh, sizeof(double) * (size_t)n0 * N, cudaMemcpyHostToDevice,
                       c->io_st));
    CK(cudaEventRecord(c->ev_h2d[0], c->io_st));
  }
  for (int r0 = 0, bi = 0; r0 < nrhs; r0 += B, ++bi) {
    const int nb = std::min(B, nrhs - r0);
    if (hio) {
      CK(cudaStreamWaitEvent(c->st, c->ev_h2d[bi & 1], 0));  // this batch's sources are on the device
      if (r0 + B < nrhs) {  // the next batch's sources travel while this batch solves
        const int nn = std::min(B, nrhs - r0 - B);
        CK(cudaMemcpyAsync(const_cast<double*>(f) + (size_t)(r0 + B) * N, hio->fh + (size_t)(r0 + B) * N,
                           sizeof(double) * (size_t)nn * N, cudaMemcpyHostToDevice, c->io_st));
        CK(cudaEventRecord(c->ev_h2d[(bi + 1) & 1], c->io_st));
      }
    }
    pt_stats sb;
    std::memset(&sb, 0, sizeof(sb));
    long long bls = 0, bii = 0, bto = 0, bla = 0, bk1l = 0;
    double btms = 0, bkms[3] = {0, 0, 0}, bk1b = 0, bcms[5] = {0, 0, 0, 0, 0}, bdfl = 0;
    double bcf[5] = {0, 0, 0, 0, 0}, bcb[5] = {0, 0, 0, 0, 0};
    std::vector<int> bh(hist.size(), 0);
    if (stats) {
      const int mi = pt_residuals_stride(cfg);
      sb.iterations = stats->iterations ? stats->iterations + r0 : nullptr;
      sb.residuals = stats->residuals ? stats->residuals + (size_t)r0 * mi : nullptr;
      sb.n_residuals = stats->n_residuals ? stats->n_residuals + r0 : nullptr;
      sb.relres = stats->relres ? stats->relres + r0 : nullptr;
      sb.converged = stats->converged ? stats->converged + r0 : nullptr;
      sb.traces = stats->traces ? stats->traces + (size_t)r0 * nO : nullptr;
      sb.polarized = stats->polarized ? stats->polarized + (size_t)r0 * 2 * nO : nullptr;
      sb.layer_solves = &bls;
      sb.inner_iters = &bii;
      sb.touches = &bto;
      sb.inner_hist = bh.empty() ? nullptr : bh.data();
      sb.inner_hist_len = (int)bh.size();
      sb.timing_ms = &btms;
      sb.kernel_ms = bkms;
      sb.k1_bytes = &bk1b;
      sb.launches = &bla;
      sb.k1_launches = &bk1l;
      sb.class_ms = bcms;
      sb.dense_flops = &bdfl;
      sb.class_flops = bcf;
      sb.class_bytes = bcb;
    }
    const int rc = solve_batch(c, f + (size_t)r0 * N, nb, cfg, u + (size_t)r0 * N, stats ? &sb : nullptr);
    if (rc != PT_OK && rc != PT_NOT_CONVERGED) {
      if (hio) cudaStreamSynchronize(c->io_st);
      return rc;
    }
    if (rc == PT_NOT_CONVERGED) worst = rc;
    if (hio) {  // this batch's wavefields travel while the next batch solves
      CK(cudaEventRecord(c->ev_done, c->st));
      CK(cudaStreamWaitEvent(c->io_st, c->ev_done, 0));
      CK(cudaMemcpyAsync(hio->uh + (size_t)r0 * N, u + (size_t)r0 * N, sizeof(double) * (size_t)nb * N,
                         cudaMemcpyDeviceToHost, c->io_st));
    }
    ls += bls, ii += bii, to += bto, la += bla, k1l += bk1l, tms += btms, k1b += bk1b, dfl += bdfl;
    for (int i = 0; i < 3; ++i) kms[i] += bkms[i];
    for (int i = 0; i < 5; ++i) {
      cms[i] += bcms[i];
      cf[i] += bcf[i];
      cb[i] += bcb[i];
    }
    for (size_t i = 0; i < hist.size(); ++i) hist[i] += bh[i];
  }
  if (stats) {
    if (stats->layer_solves) stats->layer_solves[0] = ls;
    if (stats->inner_iters) stats->inner_iters[0] = ii;
    if (stats->touches) stats->touches[0] = to;
    for (size_t i = 0; i < hist.size(); ++i) stats->inner_hist[i] = hist[i];
    if (stats->timing_ms) stats->timing_ms[0] = tms;
    if (stats->kernel_ms)
      for (int i = 0; i < 3; ++i) stats->kernel_ms[i] = kms[i];
    if (stats->k1_bytes) stats->k1_bytes[0] = k1b;
    if (stats->launches) stats->launches[0] = la;
    if (stats->k1_launches) stats->k1_launches[0] = k1l;
    if (stats->class_ms)
      for (int i = 0; i < 5; ++i) stats->class_ms[i] = cms[i];
    if (stats->dense_flops) stats->dense_flops[0] = dfl;
    if (stats->class_flops)
      for (int i = 0; i < 5; ++i) stats->class_flops[i] = cf[i];
    if (stats->class_bytes)
      for (int i = 0; i < 5; ++i) stats->class_bytes[i] = cb[i];
  }
  if (hio) CK(cudaStreamSynchronize(c->io_st));
  if (worst != PT_OK) g_err = "outer GMRES did not reach ktol within max_iter";
  return worst;
}

int pt_solve(pt_ctx* c, const double* f, int nrhs, const pt_krylov* cfg, double* u, pt_stats* stats) {
  if (!c || !f || !u || !cfg || nrhs <= 0) return PT_BAD_ARGUMENT;
  CK(cudaSetDevice(c->dev));
  const size_t bytes = sizeof(double2) * (size_t)nrhs * c->wz * c->wx;
  if (bytes > c->io_bytes) {
    if (c->io_f) cudaFree(c->io_f);
    if (c->io_u) cudaFree(c->io_u);
    c->io_f = c->io_u = nullptr;
    CK(cudaMalloc(&c->io_f, bytes));
    CK(cudaMalloc(&c->io_u, bytes));
    c->io_bytes = bytes;
  }
  double2 *fd = c->io_f, *ud = c->io_u;
  if (nrhs > batch_rhs(c)) {  // several lockstep batches: host copies of the neighbouring batches overlap each solve
    const HostIO hio{f, u};
    return solve_batches(c, reinterpret_cast<const double*>(fd), nrhs, cfg, reinterpret_cast<double*>(ud), stats, &hio);
  }
  CK(cudaMemcpyAsync(fd, f, bytes, cudaMemcpyHostToDevice, c->st));
  int rc = pt_solve_device(c, reinterpret_cast<const double*>(fd), nrhs, cfg, reinterpret_cast<double*>(ud), stats);
  cudaError_t e = cudaMemcpyAsync(u, ud, bytes, cudaMemcpyDeviceToHost, c->st);
  cudaStreamSynchronize(c->st);
  if (e != cudaSuccess && rc == PT_OK) {
    g_err = cudaGetErrorString(e);
    return PT_CUDA_ERROR;
  }
  return rc;
}

int pt_layer_solve(pt_ctx* c, int layer, const double* rhs, int nrhs, double inner_ktol, int inner_max_iter,
                   double* out, pt_stats* stats) {
  if (!c || layer < 0 || layer >= c->L || nrhs <= 0) return PT_BAD_ARGUMENT;
  CK(cudaSetDevice(c->dev));
  Stage S;
  OJob j = blank_job(layer);
  j.vol = 1;
  j.vfull = 1;
  j.nout = -1;
  for (int r = 0; r < 1; ++r) S.jobs.push_back(j);
  if (finalize_stage(c, S)) return PT_CUDA_ERROR;
  if (ensure_scratch(c, nrhs, 1)) return PT_CUDA_ERROR;
  const LayerInfo& li = c->lay[layer];
  const long long N = (long long)li.w * c->wx;
  const size_t bytes = sizeof(double2) * (size_t)nrhs * N;
  double2 *fd = nullptr, *ud = nullptr;
  CK(cudaMalloc(&fd, bytes));
  CK(cudaMalloc(&ud, bytes));
  CK(cudaMemcpy(fd, rhs, bytes, cudaMemcpyHostToDevice));
  CK(cudaMemset(c->err_d, 0, sizeof(int)));
  CK(cudaMemset(c->cnt_d, 0, sizeof(unsigned long long) * 4));
  CK(cudaMemset(c->hist_d, 0, sizeof(int) * PT_HIST));
  std::vector<int> all(nrhs);
  for (int r = 0; r < nrhs; ++r) all[r] = r;
  int rc = set_active(c, all);
  SolveIO io{fd, N, ud, N, inner_ktol, inner_max_iter};
  VecView dummy{c->TR, c->nO};
  if (!rc) rc = run_stage(c, S, VecTab{{dummy, dummy, dummy}}, nrhs, io);
  CK(cudaStreamSynchronize(c->st));
  CK(cudaMemcpy(out, ud, bytes, cudaMemcpyDeviceToHost));
  int ecode = 0;
  check_err(c, &ecode);
  if (stats) {
    unsigned long long cnt[4] = {0, 0, 0, 0};
    CK(cudaMemcpy(cnt, c->cnt_d, sizeof(cnt), cudaMemcpyDeviceToHost));
    if (stats->inner_iters) stats->inner_iters[0] = (long long)cnt[0];
    if (stats->touches) stats->touches[0] = (long long)cnt[1] + c->touch_extra;
    if (stats->inner_hist && stats->inner_hist_len > 0) {
      int hh[PT_HIST];
      CK(cudaMemcpy(hh, c->hist_d, sizeof(hh), cudaMemcpyDeviceToHost));
      for (int i = 0; i < stats->inner_hist_len; ++i) stats->inner_hist[i] = i < PT_HIST ? hh[i] : 0;
    }
  }
  cudaFree(fd);
  cudaFree(ud);
  for (auto& kv : S.tasks) cudaFree(kv.second.d);
  cudaFree(S.jobs_d);
  cudaFree(S.stage_jobs_d);
  cudaFree(S.ljobs_d);
  if (rc) return rc;
  return ecode;
}

// K1 alone on device-resident volumes: x = H_c^{-1} b for nrhs right-hand sides [nrhs][wz_c][w], on the
// context's stream (synchronised before returning).  The offline stage builds the Green blocks and the
// operators of the online restructuring through this entry (offline.py, green.py:103-129 as many-RHS solves).
int pt_cell_solve_device(pt_ctx* c, int layer, int cell, const double* b_dev, int nrhs, double* x_dev) {
  if (!c || !b_dev || !x_dev || layer < 0 || layer >= c->L || cell < 0 || cell >= c->Lc || nrhs <= 0)
    return PT_BAD_ARGUMENT;
  CK(cudaSetDevice(c->dev));
  const CellInfo& ci = c->cel[layer * c->Lc + cell];
  double2* bd = reinterpret_cast<double2*>(const_cast<double*>(b_dev));
  double2* xd = reinterpret_cast<double2*>(x_dev);
  std::vector<K1Task> tasks;
  long long z = 0;
  // 8 columns per cluster pair (the DMMA path) where K1's epilogue holds them (8 w <= 4 K1_CONSUMERS), else 4
  const int nc = std::getenv("PT_K1_NC") ? atoi(std::getenv("PT_K1_NC")) : (8 * c->wmax <= 4 * K1_CONSUMERS ? 8 : 4);
  for (int q0 = 0; q0 < nrhs; q0 += nc) {  // one cluster pair per nc columns (cm = 1)
    K1Task t;
    t.cell = layer * c->Lc + cell;
    t.jb = 0;
    t.q0 = q0;
    t.nq = std::min(nc, nrhs - q0);
    t.zoff = z;
    z += (long long)ci.wzc * ci.w * nc;
    tasks.push_back(t);
  }
  K1Task* td = nullptr;
  if (upload(&td, tasks.data(), tasks.size())) return PT_CUDA_ERROR;
  if (ensure_z(c, z)) return PT_CUDA_ERROR;
  K1Params kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.cells = c->cel_d;
  kp.layers = c->lay_d;
  kp.tasks = td;
  kp.sinv = c->sinv_d;
  kp.lz = c->lz_d;
  kp.uz = c->uz_d;
  kp.R = nrhs;
  kp.pass = 2;
  kp.npml = c->npml;
  kp.wx = c->wx;
  kp.Lc = c->Lc;
  kp.wmax = c->wmax;
  kp.slot_bytes = c->slot_bytes;
  kp.ns = c->ns;
  kp.cm = 1;
  kp.Z = c->Z;
  kp.dbg = std::getenv("PT_K1_DBG") ? atoi(std::getenv("PT_K1_DBG")) : 0;
  {
    static long long* tprof_d2 = nullptr;
    if (std::getenv("PT_K1_TPROF") && !tprof_d2) cudaMalloc(&tprof_d2, 6 * sizeof(long long));
    kp.tprof = std::getenv("PT_K1_TPROF") ? tprof_d2 : nullptr;
  }
  kp.bd = bd;
  kp.xd = xd;
  const bool timed = kp.tprof != nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (timed) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c->st);
  }
  CK(k1_launch(kp, (int)tasks.size(), nc, c->wmax, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (timed) {  // PT_K1_TPROF: launch time and the per-phase clock64 totals of CTA 0
    cudaEventRecord(e1, c->st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    long long tt[6];
    cudaMemcpy(tt, kp.tprof, sizeof(tt), cudaMemcpyDeviceToHost);
    fprintf(stderr, "cell_solve nc=%d tasks=%d dbg=%d: %.1f us | prologue %lld preload %lld bar1 %lld matvec %lld "
            "bar2 %lld epi %lld\n", nc, (int)tasks.size(), kp.dbg, ms * 1e3f, tt[0], tt[1], tt[2], tt[3], tt[4], tt[5]);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  cudaFree(td);
  return PT_OK;
}

int pt_cell_solve(pt_ctx* c, int layer, int cell, const double* b, int nrhs, double* x) {
  if (!c || !b || !x || layer < 0 || layer >= c->L || cell < 0 || cell >= c->Lc || nrhs <= 0) return PT_BAD_ARGUMENT;
  CK(cudaSetDevice(c->dev));
  const CellInfo& ci = c->cel[layer * c->Lc + cell];
  const size_t bytes = sizeof(double2) * (size_t)nrhs * ci.wzc * ci.w;
  double2 *bd = nullptr, *xd = nullptr;
  CK(cudaMalloc(&bd, bytes));
  if (cudaMalloc(&xd, bytes) != cudaSuccess) {
    cudaFree(bd);
    g_err = "pt_cell_solve: out of device memory";
    return PT_CUDA_ERROR;
  }
  int rc = cudaMemcpy(bd, b, bytes, cudaMemcpyHostToDevice) == cudaSuccess ? PT_OK : PT_CUDA_ERROR;
  if (rc == PT_OK)
    rc = pt_cell_solve_device(c, layer, cell, reinterpret_cast<const double*>(bd), nrhs, reinterpret_cast<double*>(xd));
  if (rc == PT_OK && cudaMemcpy(x, xd, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) rc = PT_CUDA_ERROR;
  cudaFree(bd);
  cudaFree(xd);
  return rc;
}

}  // extern "C"
