// Kernel parameter blocks and launchers shared by the kernels and the host
// orchestration (solver.cu).
#pragma once
#include "pt_device.cuh"

#define INNER_NC 8

#include <unordered_map>
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs more than it was given so far:
// the attribute calls cost microseconds of host time per launch otherwise
inline void set_smem_attr(const void* fn, size_t bytes) {
  static std::unordered_map<const void*, size_t> done;
  size_t& v = done[fn];
  if (bytes > v) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    v = bytes;
  }
}
#define INNER_CS 8  // CTAs per inner-GMRES cluster (portable cluster size)
#define PT_HIST 64

struct VecView {
  double2* p;
  long long stride;
};
struct VecTab {
  VecView v[3];  // 0 IN, 1 OUT, 2 AUX
};

struct K1Params {
  int jc8;                // DMMA path (NC = 8): columns per ring chunk (multiple of 4; K1_JC8 or PT_K1_JC8)
  const CellInfo* cells;
  const LayerInfo* layers;
  const OJob* jobs;
  const int* ljobs;
  const K1Task* tasks;
  const double2* sinv;
  const double2* lz;
  const double2* uz;
  int R, pass, npml, wx, Lc, wmax;
  int slot_bytes, ns;
  int cm;             // column CTAs per half-chain (cluster = 2*cm CTAs, factor chunks multicast)
  const double2* f;
  long long f_stride;
  const double2* P;   // [job][4][R][wx]
  const double2* tr;  // [job][R][Lc-1][2][wmax]
  double2* tables;    // [job][Lc][4][R][wmax]
  double2* smp;       // [job][4][R][wx]
  double2* u;
  long long u_stride;
  double2* Z;
  const double2* bd;  // pass 2 (dense test mode): b [q][wzc][w]
  double2* xd;        // pass 2: x [q][wzc][w]
  // pass 0 of a volume-source stage: [layer][R] 1 = the RHS's split source is nonzero somewhere in the layer
  // (k_slab_flags); a task whose columns all have a zero source and no panels writes zero outputs and exits
  // (point / surface sources touch one layer of L).  NULL: no shortcut.
  const int* zflag;
  long long* tprof;   // optional per-phase clock64 totals of CTA 0 (debug instrumentation)
  int dbg;            // debug: 1 = no factor streaming (timing only), 2 = no matvec (timing only)
  int s0;             // pass 0 also writes the layer-row samples of its solution into smp
};

struct InnerParams {
  const CellInfo* cells;
  const LayerInfo* layers;
  const OJob* jobs;
  const int* stage_jobs;  // job id per CTA
  const double2* green;
  const double2* dense;   // dense inner operators (LayerInfo.dense_off), or null: item programs
  long long coop_region;  // cooperative kernel: bytes of its shared-memory ring (set by the launcher)
  // fused sample-only stage (cooperative kernel): gather -> pass-0 product -> inner -> sampled trace
  // response -> combine in one launch (stage_dev.cuh bodies); fused = 0: inner GMRES only
  int fused;
  VecTab tab;
  const int* rmap;
  int wx, ngl, maxj, kmax;
  double2* P;
  double2* smp;
  const double2* q0;
  const double2* gsmp;
  const int* grp;
  const int* ljobs;
  const IItem* items;
  const int* op_ph;       // phase begin offsets into items (op_nph + 1 entries)
  int op_nph;
  const int* pre_ph;
  int pre_nph;
  int R, Lc, wmax, cap, max_iter;
  double ktol;
  const double2* tables;  // [job][Lc][4][R][wmax]
  double2* tr;            // [job][R][Lc-1][2][wmax]
  double2* scratch;       // per (job, r): (cap + 5) vectors of nmax
  long long inst_stride, nmax;
  double2* hess;
  long long hstride;
  int* iters;             // [job][R] inner iterations (-1 = error)
  int* state;             // [job][R] 0 running, 1 converged, 2 failed (cluster-shared)
  double* beta0;          // [job][R] initial preconditioned residual norms
  int* err;               // PT_* code (atomicMax)
  unsigned long long* counters;  // [0] inner iterations, [1] Green touches, [2] instances
  int* hist;              // [PT_HIST] histogram of inner iteration counts
  long long op_blocks, pre_blocks;  // block matvecs per inner op / preconditioner application
  int tprof;              // debug: accumulate clock64 segment totals of CTA 0 (PT_INNER_TPROF)
  int nitems;             // op + pre program items (staged in shared memory)
  int mg;                 // 8-row Green tiles per work group (inner_mg(wmax))
  int tring;              // Green-tile ring slots of the item-program path (inner_tring)
  int coop_sms;           // SMs (CTAs) of the cooperative inner kernels; 0 = all
  int sstep;              // dense stack [pre; E pre; E^2 pre] present: s-step start of the inner GMRES
  int rhs_ready;          // the stage's producer (pass-0 product) wrote rhs_pol into the VB scratch vectors
  int unit_major;         // dense products: unit-major work split instead of tile-major (PT_UNIT_MAJOR)
  int da_slot;            // cooperative dense passes: ring slot capacity in bytes (set by the launcher; 0 = default)
  int tprefetch;          // item-program kernel: next phase's first Green tiles issued before the grid barrier
  int arn_fast;           // Arnoldi steps of small instances with the basis prefetched (PT_ARN_SLOW = 0)
  // whole-GPU item-program kernel (inner_items.cu): RHS-minor scratch [job][vector][n-tile][nmax][8]
  long long s2_vec, s2_job;  // double2 strides of one vector / one job (set by the launcher)
  double2* part;             // vector-phase partials [3][part_items][cap + 2][8]
  long long part_items;
  // scan form of the preconditioner program (single-job stages; solver.cu build_inner): op items + scan pre items
  const IItem* items_px;
  const int* pre_ph_px;
  int pre_nph_px, nitems_px;
  int ii_dbg;                // PT_II_DBG timing switches of inner_items.cu (results invalid when set)
  int ii_tilecost;           // PT_II_TILECOST: fixed cycles per CTA tile in the tile-shape cost model (0 = 3000)
  int ii_trace;              // PT_II_TRACE: event trace of CTA (ii_trace - 1), thread 0
};

size_t k1_smem_bytes(int wmax, int nc, int slot_bytes, int ns);
cudaError_t k1_launch(const K1Params& p, int ntasks, int nc, int wmax, cudaStream_t st);
#define K1_CONSUMERS 224  // 7 consumer warps + 1 producer warp: 8 warps keep 255 registers per thread
#define K1_THREADS (K1_CONSUMERS + 32)
#define K1_NS 8       // ring slots (multiple of every multicast group size)
#define K1_NS_LOG2 3
#define K1_RW 4       // rows per lane in the K1 matvec: cell width w <= 128
#define K1_DMMA_ITEMS 3  // 8-row tiles per warp in the DMMA path: ceil(128/8) <= 3*7
// DFMA path: columns per consumer warp per ring chunk (7 warps per chunk)
__host__ __device__ constexpr int k1_jw(int nc) { return nc == 1 ? 5 : (nc == 2 ? 4 : 2); }
#define K1_JC8 12        // narrowest ring chunk width (columns) of the DMMA path: 3 k-steps (k1_launch widens it)
size_t inner_smem_bytes(int wmax, int nitems, int tring);
int inner_tring(int wmax, int nitems);
int inner_mg(int wmax);
cudaError_t inner_launch(const InnerParams& p, int njobs, cudaStream_t st);
// whole-GPU cooperative inner GMRES (dense operators); cudaErrorNotSupported: use inner_launch
cudaError_t inner_coop_launch(const InnerParams& p, int njobs, cudaStream_t st);
int inner_coop_max_units();  // (job, 8-RHS group) units one cooperative inner launch holds
// whole-GPU inner GMRES over the item programs with all RHS of a job per tensor-core tile (inner_items.cu);
// cudaErrorNotSupported: outside its limits (caller falls back)
cudaError_t inner_items_launch(const InnerParams& p, int njobs, cudaStream_t st);
long long inner_items_part_items(int num_sms, int jmax, int rmax);  // partial records the launcher needs
void inner_tprof_dump(const char* tag);
__global__ void k_dense_tiles(const double2* src, double2* dst, int n, int kc);
__global__ void k_dense_tiles_stack3(const double2* s0, const double2* s1, const double2* s2, double2* dst, int n,
                                     int kc);
#define DA_KC 8  // k-steps per dense-apply chunk (inner_gmres.cu; the stored fragment layout depends on it)
// double2 size of one stored dense inner matrix (k_dense_tiles layout)
__host__ __device__ inline long long dense_matrix_elems(long long n) {
  const long long T8 = (n + 7) / 8, nks = n / 4, nch = (nks + DA_KC - 1) / DA_KC;
  return nch * T8 * DA_KC * 32;
}
// first layer-solve pass (no volume source) as a dense product with the offline pass-0 operators
// Optional second output of the pass-0 product: the inner GMRES rhs_pol (sie.py:230-242, negated Newton rows
// n, n+1 of cell I and 0, 1 of cell I+1) written straight into each instance's inner scratch vector, so the
// inner kernel needs no gather pass: element e of instance (job, q) at base + (job R + q) stride + off + e.
struct RhsOut {
  double2* base;
  long long stride, off;
};

cudaError_t pass0_launch(const int* grp, int ngroups, const int* ljobs, const OJob* jobs, const CellInfo* cells,
                         const LayerInfo* layers, const double2* q0, const double2* P, double2* tables, double2* smp,
                         int R, int Lc, int wx, int wmax, int kmax, int max_jobs_per_layer, cudaStream_t st,
                         int accum = 0, const VecTab* tab = nullptr, const int* rmap = nullptr,
                         const RhsOut* rhs_out = nullptr);  // PT_INNER_TPROF: print and reset CTA 0's segment clocks
// smp += trace-source response (sampled Green rows) for every (job, cell, output row, RHS)
cudaError_t green_samples_launch(const OJob* jobs, int J, const CellInfo* cells, const LayerInfo* layers,
                                 const double2* gsmp, const double2* tr, double2* smp, int R, int Lc, int wx,
                                 int wmax, int kmax, int num_sms, cudaStream_t st, const VecTab* tab = nullptr,
                                 const int* rmap = nullptr);

// many-RHS forms of the two products above as one streaming tensor-core GEMM kernel (stage_gemm.cu)
int stage_gemm_min_cols(int mode);  // mode 0: sampled response, 1: pass-0 product
cudaError_t sample_gemm_launch(const OJob* jobs, int J, const CellInfo* cells, const LayerInfo* layers,
                               const double2* gsmp, const double2* tr, double2* smp, int R, int Lc, int wx, int wmax,
                               int kmax, int num_sms, cudaStream_t st, const VecTab* tab, const int* rmap);
cudaError_t pass0_gemm_launch(const int* grp, int ngroups, const int* ljobs, const OJob* jobs, const CellInfo* cells,
                              const LayerInfo* layers, const double2* q0, const double2* P, double2* tables,
                              double2* smp, int R, int Lc, int wx, int wmax, int kmax, int max_jobs_per_layer,
                              int num_sms, cudaStream_t st, int accum, const RhsOut* rhs_out);

__global__ void k_gather_panels(const OJob* jobs, int njobs, VecTab t, const int* rmap, int nq, int wx,
                                double2* P);
__global__ void k_combine(const OJob* jobs, int njobs, VecTab t, const int* rmap, int nq, int wx,
                          const double2* smp);
__global__ void k_lincomb(VecView dst, long long doff, VecView xv, long long xoff, double a, VecView yv,
                          long long yoff, double b, int use_y, long long len, const int* rmap, int nq);
__global__ void k_norm2(VecView v, long long len, const int* rmap, double* out);
__global__ void k_inner_lu(const int* __restrict__ stage_jobs, const OJob* __restrict__ jobs,
                           const LayerInfo* __restrict__ layers, const double2* __restrict__ lu,
                           const double2* __restrict__ tables, double2* __restrict__ trc, int R, int Lc, int wmax,
                           unsigned long long* counters);
__global__ void k_cdot(VecView x, VecView y, long long len, const int* rmap, double2* out);
__global__ void k_bicg_update(int mode, VecView d, VecView x, VecView y, VecView z, const double2* a,
                              const double2* b, long long len, const int* rmap, int nq);
__global__ void k_scale_div(VecView dst, VecView src, long long len, const int* rmap, int nq,
                            const double* scale);
__global__ void k_arnoldi(double2* V, long long vstride, long long n, int j, const int* rmap, double2* hout,
                          int hld);
__global__ void k_arnoldi2(double2* V, long long vstride, long long n, int j, const int* rmap, double2* hout,
                           int hld);
__global__ void k_accum_x(VecView x, const double2* V, long long vstride, long long n, const double2* y,
                          int yld, int k, const int* rmap, int nq);
__global__ void k_residual(const double2* u, const double2* f, long long stride, int wz, int wx, const double2* tx,
                           const double2* tz, const double* m, double omega2, const int* rmap, double* out,
                           const double2* hdiag);
__global__ void k_slab_flags(const double2* f, long long stride, const LayerInfo* layers, int wx, int R, int* flags);
__global__ void k_vol_norm2(const double2* f, long long stride, long long N, double* out);
__global__ void k_green_tiles(const double2* src, double2* dst, int w, int nb);
__global__ void k_block2_mm(const double2* A, const double2* B, double2* C, int w);
__global__ void k_q0_rows(const double2* src, double2* dst, int w, int nk, int K);
