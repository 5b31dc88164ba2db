/*
 * pt_b200.h -- C ABI of the B200-native online stage of the nested
 * polarized-traces Helmholtz solver (libpt_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary.
 * Complex numbers are interleaved (re, im) doubles, i.e. numpy complex128 /
 * C99 double _Complex / CUDA double2.
 *
 * What each entry point replaces in the reference
 * (/root/reference/pkg/src/polartraces):
 *
 *   pt_create       build_nested_layers(..., backend="pt") + PolarizedTracesSolver.__init__
 *                   (nested.py:507-521, sie.py:368-381): the offline factors computed by the
 *                   host (paper_1510_01831_b200/offline.py) are uploaded once.
 *   pt_solve        PolarizedTracesSolver.solve (sie.py:392-439) for nrhs sources at once,
 *                   host buffers in and out (the call a ctypes/cffi binding makes).
 *   pt_solve_device the same with device-resident f/u (e.g. torch CUDA tensors).
 *   pt_layer_solve  NestedLayerSolver.solve (nested.py:344-353), one layer, nrhs volumes:
 *                   the "layer object" protocol of sie.py:112-118 (test/plugin hook).
 *   pt_cell_solve   LayerWorkspace.solve on one cell (subdomain.py:214-221 -> SuperLU
 *                   solve): the K1 kernel alone (test hook); pt_cell_solve_device: the same on
 *                   device buffers, the many-RHS solves of the offline stage (green.py:103-129).
 *   pt_set_stream / pt_set_profiling: run on a caller stream (e.g. torch's) / time every launch.
 *   pt_residuals_stride: per-RHS length of the residual-history buffer for a Krylov config.
 *   pt_destroy / pt_last_error / pt_version.
 *
 * Return codes (errors map to the reference's exceptions, sie.py:420-425,
 * nested.py:148-152, krylov.py:101-123, subdomain.py:219-220):
 *   PT_OK 0, PT_NOT_CONVERGED 1 (KrylovBreakdown: outer did not reach ktol),
 *   PT_INNER_NOT_CONVERGED 2 (InnerSolveError), PT_BREAKDOWN 3 (KrylovBreakdown:
 *   zero Hessenberg column / happy breakdown before convergence), PT_BAD_ARGUMENT 4
 *   (ValueError), PT_CAPACITY 5 (a Krylov basis outgrew its preallocated capacity),
 *   PT_CUDA_ERROR -1 (see pt_last_error).
 */
#ifndef PT_B200_H
#define PT_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define PT_OK 0
#define PT_NOT_CONVERGED 1
#define PT_INNER_NOT_CONVERGED 2
#define PT_BREAKDOWN 3
#define PT_BAD_ARGUMENT 4
#define PT_CAPACITY 5
#define PT_CUDA_ERROR (-1)

typedef struct pt_ctx pt_ctx;

/* Problem geometry and offline factors.  All arrays may be host or device
 * pointers (copied with cudaMemcpyDefault); the caller keeps ownership. */
typedef struct {
  int nx, nz, npml;          /* interior nodes and PML width (Grid, discretization.py:58-71) */
  int L, Lc;                 /* layers and cells per layer */
  double h, omega;
  const int* layer_extents;  /* [L]  partition_layers extents (subdomain.py:93-100) */
  const int* cell_extents;   /* [Lc] swapped-frame cell extents (nested.py:294-296) */
  /* global 5-point operator for the true residual (sie.py:441-445) */
  const double* tx;          /* [3][wx] complex: lower, main, upper of T_x */
  const double* tz;          /* [3][wz] complex: lower, main, upper of T_z */
  const double* m;           /* [wz][wx] real squared slowness */
  /* layer-level slot sources (subdomain.py:157-182): coefficient of v0,v1,vn,vnp */
  const double* layer_coefs; /* [L][4] complex */
  /* per cell, layer-major (id = l*Lc + c) */
  const double* cell_coefs;  /* [L*Lc][4] complex, cell-level slot coefficients */
  const double* const* lz;   /* [L*Lc] -> [wz_c] complex block sub-diagonal scalars  */
  const double* const* uz;   /* [L*Lc] -> [wz_c] complex block super-diagonal scalars */
  const double* const* sinv; /* [L*Lc] -> [wz_c][w][w] complex Schur inverses, column-major blocks */
  const double* const* green;/* [L*Lc] -> [4 rows][4 slots][w][w] complex, column-major blocks; NULL = a
                              * factor-only context for pt_cell_solve(_device) (the offline stage) */
  /* optional (NULL: sampled outputs come from a second cell-solve pass):
   * [L*Lc] -> [wz_c][4 layer trace rows 0,1,n,n+1][4 slots][w] complex, the trace-source
   * response H_c^{-1}(coef_s E_krow_s) sampled at every block row and the layer trace rows */
  const double* const* gsmp;
  /* optional (NULL: layer solves without a volume source run the first cell-solve pass):
   * [L*Lc] -> [M][4 nk4] complex row-major, the cell response to the layer slot sources
   * (coef_s E at layer row prow_s, every kept block row k; nk = kept rows, nk4 = roundup(nk, 4))
   * sampled at the Newton-table block rows (4 x w) and the layer trace rows of every kept block
   * row (4 nk); M = roundup(4 w + 4 nk, 8) */
  const double* const* q0;
  /* optional (NULL: the inner GMRES applies its operator and preconditioner panel by panel):
   * [L] -> [inner_dense_count][n][n] complex row-major, n = 4 (Lc-1) w: the layer's inner GS
   * preconditioner and preconditioned operator pre(op(.)) as dense matrices (sie.py:203-329), then
   * optionally E pre and E^2 pre (E = pre(op(.)) - I) for the s-step start of the inner GMRES */
  const double* const* inner_dense;
  /* optional (NULL: the inner solve is the polarized-traces GMRES of nested.py:125-153):
   * [L] -> [m][m] complex row-major, m = 2 (Lc-1) w: the inverse of the assembled cell-interface
   * system of the direct inner backend (backend="lu", nested.py:156-254); the inner solve of a layer
   * solve is then x = A^-1 b with b = (row n of cell i, row 1 of cell i+1) of the Newton tables */
  const double* const* inner_lu;
  /* 1: the reference's factored boundary pipeline (assembled_boundary=True, nested.py:355-486) is
   * selected.  The sample-only layer solves run the same linear maps either way (pass-0 operator =
   * M_f + direct part, sampled trace response = M_u); this selects its TouchCounter accounting:
   * per boundary_samples call sum_c 16 w s_c + 16 s_c^2 + 4 nslot_c s_c w (s_c = kept rows of cell c) */
  int assembled_boundary;
  int inner_dense_count;     /* matrices per layer in inner_dense: 2, or 4 with the s-step operators */
  /* optional (NULL: Tx_main + Tz_main - omega^2 m): [wz][wx] complex diagonal of the global operator used by
   * the true residual, for a caller-supplied global_operator (sie.py:381, 387-390); the neighbour couplings
   * are tx / tz's lower and upper diagonals either way */
  const double* hdiag;
} pt_problem;

typedef struct {
  double ktol;           /* outer relative preconditioned residual (KrylovConfig.ktol) */
  int max_iter;          /* KrylovConfig.max_iter */
  int restart;           /* KrylovConfig.restart (0 = none) */
  double inner_ktol;     /* NestedLayerSolver inner_ktol (1e-6) */
  int inner_max_iter;    /* NestedLayerSolver inner_max_iter (200) */
  int precond;           /* 0 = "gs", 1 = "jac" (sie.py:407) */
  int method;            /* 0 = "gmres" (krylov.py:53-135), 1 = "bicgstab" (krylov.py:138-201) */
} pt_krylov;

typedef struct {
  /* all optional (NULL = not requested); sized by the caller */
  double* iterations;    /* [nrhs] outer GMRES iterations (float, krylov.py:135) */
  double* residuals;     /* [nrhs][pt_residuals_stride(cfg)] residual history (relative preconditioned) */
  int* n_residuals;      /* [nrhs] entries written per rhs */
  double* relres;        /* [nrhs] ||H u - f|| / ||f|| */
  int* converged;        /* [nrhs] */
  double* traces;        /* [nrhs][nI][2][wx] complex reassembled traces (down + up) */
  double* polarized;     /* [nrhs][4*nI*wx] complex polarized solution */
  long long* layer_solves;   /* [1] number of layer-solve instances executed */
  long long* inner_iters;    /* [1] sum of inner GMRES iterations over all instances */
  long long* touches;        /* [1] inner Green-block element touches (TouchCounter.total) */
  int* inner_hist;           /* [inner_hist_len] histogram of inner iteration counts */
  int inner_hist_len;
  double* timing_ms;         /* [1] device time of the online solve (CUDA events) */
  /* profiling (filled when pt_set_profiling(ctx, 1)): CUDA events around every launch */
  double* kernel_ms;         /* [3] summed device time: K1 cell solves, inner GMRES, other kernels */
  double* k1_bytes;          /* [1] algorithmic S^-1 bytes of all K1 launches: 32*wz_c*w_c^2 per cell solve */
  long long* launches;       /* [1] kernels launched by this solve */
  long long* k1_launches;    /* [1] K1 launches */
  double* class_ms;          /* [5] device time per launch class: K1, inner GMRES, glue, sampled trace
                                response, pass-0 product (profiling only) */
  double* dense_flops;       /* [1] algorithmic flops of the dense inner products: 8 n^2 per instance per product */
  /* executed work per launch class (same classes as class_ms): flops = 8 per complex multiply-add the kernels
   * perform (inner GMRES: the TouchCounter total x 8, or the dense products), bytes = the operator data the
   * launches stream (Schur inverses, Green blocks, pass-0 and sampled-response operators) */
  double* class_flops;       /* [5] */
  double* class_bytes;       /* [5] */
} pt_stats;

int pt_create(const pt_problem* prob, int device, pt_ctx** out);
/* run subsequent work on a caller-owned cudaStream_t (NULL = the context's own stream) */
int pt_set_stream(pt_ctx* ctx, void* stream);
/* 1 = bracket every launch with CUDA events and report per-kernel-class times in pt_stats */
int pt_set_profiling(pt_ctx* ctx, int enable);
int pt_destroy(pt_ctx* ctx);

int pt_solve(pt_ctx* ctx, const double* f, int nrhs, const pt_krylov* cfg, double* u,
             pt_stats* stats);
int pt_solve_device(pt_ctx* ctx, const double* f_dev, int nrhs, const pt_krylov* cfg,
                    double* u_dev, pt_stats* stats);

/* layer ell (0-based): u_l = (H_l)^{-1} rhs for nrhs slabs [nrhs][n_l+2npml][wx] (host) */
int pt_layer_solve(pt_ctx* ctx, int layer, const double* rhs, int nrhs, double inner_ktol,
                   int inner_max_iter, double* out, pt_stats* stats);
/* cell (layer, c): x = H_c^{-1} b for nrhs right-hand sides [nrhs][wz_c][w] (host) */
int pt_cell_solve(pt_ctx* ctx, int layer, int cell, const double* b, int nrhs, double* x);
/* the same with device-resident b / x (K1 on the context's stream, synchronised on return).  The offline stage
 * runs GreenBlockSet.build (green.py:103-129, nested.py:296-307: 4 w unit-source solves per cell) and the
 * pass-0 / sampled-response operators through this entry on a factor-only context (pt_problem.green == NULL) */
int pt_cell_solve_device(pt_ctx* ctx, int layer, int cell, const double* b_dev, int nrhs, double* x_dev);

/* entries per RHS of pt_stats.residuals: max_iter + 1 for GMRES (krylov.py:53-135), 2 max_iter + 1 for
 * BiCGstab (krylov.py:138-201: the initial 1.0 plus two half steps per iteration) */
int pt_residuals_stride(const pt_krylov* cfg);

const char* pt_last_error(void);
const char* pt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PT_B200_H */
