// Outer-level kernels: equivalent-source panel gather, sample combination,
// polarized-vector algebra, fused MGS Arnoldi, and the true residual (K5).
//
// Outer vectors are RHS-major: element e of RHS r of view V lives at
// V.p[r * V.stride + e]; panels (segments) are wx long.  Stage kernels run on
// the compacted list of still-active RHS (rmap), so converged right-hand sides
// cost nothing and never feed garbage into an inner solve.
#include "pt_device.cuh"

#include <algorithm>

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

__global__ void __launch_bounds__(P0_KQ * 32) k_pass0(const int* __restrict__ grp, const int* __restrict__ ljobs,
                                                      const OJob* __restrict__ jobs,
                                                      const CellInfo* __restrict__ cells,
                                                      const LayerInfo* __restrict__ layers,
                                                      const double2* __restrict__ q0, const double2* __restrict__ P,
                                                      double2* __restrict__ tables, double2* __restrict__ smp, int R,
                                                      int Lc, int wx, int wmax, int accum, VecTab tab,
                                                      const int* rmap, int direct) {
  __shared__ double part[(P0_KQ - 1) * 2 * 4 * 32];
  pass0_item(grp, ljobs, jobs, cells, layers, q0, P, tables, smp, R, Lc, wx, wmax, blockIdx.x / Lc,
             blockIdx.x % Lc, blockIdx.y, blockIdx.z, threadIdx.x >> 5, part, 1, accum, direct ? &tab : nullptr,
             rmap);
}

__global__ void __launch_bounds__(GS_WARPS * 32) k_green_samples(
    const OJob* __restrict__ jobs, const CellInfo* __restrict__ cells, const LayerInfo* __restrict__ layers,
    const double2* __restrict__ gsmp, const double2* __restrict__ tr, double2* __restrict__ smp, int R, int Lc, int wx,
    int wmax, VecTab tab, const int* rmap, int fuse_combine) {
  extern __shared__ double2 trs[];  // [4 slots][w4][8 rhs]
  green_item(jobs, cells, layers, gsmp, tr, smp, R, Lc, wx, wmax, blockIdx.x, blockIdx.y, blockIdx.z, trs,
             fuse_combine ? &tab : nullptr, rmap);
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

// dst = src / scale[r] (scale on device)
__global__ void k_scale_div(VecView dst, VecView src, long long len, const int* rmap, int nq,
                            const double* scale) {
  const long long total = len * nq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / len);
    const long long i = e - (long long)q * len;
    const int r = rmap[q];
    const double s = scale[r];
    const double2 a = src.p[r * src.stride + i];
    dst.p[r * dst.stride + i] = make_double2(a.x / s, a.y / s);
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
                           const double2* tz, const double* m, double omega2, const int* rmap, double* out) {
  __shared__ double red[32];
  const int r = rmap[blockIdx.y];
  const double2* ur = u + r * stride;
  const double2* fr = f + r * stride;
  double rr = 0.0, ff = 0.0;
  const long long N = (long long)wz * wx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / wx), pcol = (int)(e % wx);
    // diag = (Tx_main + Tz_main) - omega^2 m
    const double2 dg = csub(cadd(tx[wx + pcol], tz[wz + q]), make_double2(omega2 * m[e], 0.0));
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
__global__ void k_green_tiles(const double2* src, double2* dst, int w) {
  const int nmt = (w + 7) >> 3;
  const long long total = 16LL * nmt * w * 8;
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
  (void)num_sms;
  if (J == 0 || R == 0) return cudaSuccess;
  const int gy = (R + 7) / 8;
  // rows per cell <= kmax kept block rows x 4 output rows; one 8-row tile per warp
  const int gz = (kmax * 4 + 8 * GS_WARPS - 1) / (8 * GS_WARPS);
  const size_t sm = sizeof(double2) * 4 * (size_t)((wmax + 3) & ~3) * 8;
  if (sm > 48 * 1024) set_smem_attr((const void*)k_green_samples, sm);
  k_green_samples<<<dim3(J * Lc, gy, gz), GS_WARPS * 32, sm, st>>>(jobs, cells, layers, gsmp, tr, smp, R, Lc, wx, wmax, tabv, rmap,
                                                                        fuse_combine);
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
                         int accum, const VecTab* tab, const int* rmap) {
  if (ngroups == 0 || R == 0) return cudaSuccess;
  const VecTab tabv = tab ? *tab : VecTab{};
  const int mp = (4 * wmax + 4 * kmax + 7) / 8 * 8;
  const int gz = (max_jobs_per_layer * R + P0_COLS - 1) / P0_COLS;
  k_pass0<<<dim3(ngroups * Lc, mp / 8, gz), P0_KQ * 32, 0, st>>>(grp, ljobs, jobs, cells, layers, q0, P, tables, smp,
                                                                 R, Lc, wx, wmax, accum, tabv, rmap, tab != nullptr);
  return cudaGetLastError();
}
