// Inner polarized-traces GMRES (replaces _InnerPT.solve_traces, nested.py:134-153).
//
// One thread-block CLUSTER (INNER_CS CTAs) per layer-solve job; the job's R
// right-hand-side instances advance in lockstep and are frozen individually
// when they converge, so every instance runs exactly the Krylov process of
// krylov.gmres (krylov.py:53-135): same operator (inner apply_M_polarized on
// the dense Green blocks, sie.py:203-228 / nested.py:113-122), same left GS
// preconditioner (sie.py:272-326), MGS Arnoldi with vdot, complex Givens, stop
// when |g_{j+1}|/beta0 <= inner_ktol, x = V_k y.  The data-dependent iteration
// count never leaves the device.
//
// The operator and preconditioner are executed from "item programs" built on
// the host: each item is one sampled panel = sum_slot G[cell][row][slot] @
// panel_slot + add - (sub0 + sub1), i.e. exactly the arithmetic of the
// reference's TraceSystem methods.  Items of one phase are independent: the
// (item x instance-batch x row-chunk) units of a phase are spread over the
// cluster's CTAs and phases are separated by cluster barriers
// (barrier.cluster release/acquire).  Arnoldi, Givens and the final x = V y of
// instance r run on CTA (r mod INNER_CS) only, so no cross-CTA reduction is
// needed and the reductions are deterministic.
#include <cooperative_groups.h>

#include "pt_launch.cuh"

namespace cg = cooperative_groups;

__device__ __forceinline__ double2* vecp(const InnerParams& p, int job, int r, int v) {
  return p.scratch + (size_t)(job * p.R + r) * p.inst_stride + (size_t)v * p.nmax;
}

__device__ __forceinline__ void csync() { cg::this_cluster().sync(); }

// Execute one program (list of phases) for the active instances, spread over the cluster.
// vmap: program vec ids {0:IN,1:OUT,2:AUX} -> scratch vector index.
__device__ void run_program(const InnerParams& p, int job, int layer, int w, const int* ph, int nph,
                            const int vmap[3], const int* act, int nact, double2* pan, double2* red, int q,
                            int CS) {
  const int tid = threadIdx.x;
  const int nb = (nact + INNER_NC - 1) / INNER_NC;
  for (int phz = 0; phz < nph; ++phz) {
    const int it0 = ph[phz], nit = ph[phz + 1] - it0;
    const int base = nit * nb;
    int nchunk = 1;
    if (base > 0 && base < CS) nchunk = min((CS + base - 1) / base, max(1, w / 8));
    const int units = base * nchunk;
    for (int u = q; u < units; u += CS) {
      const int ii = u / (nb * nchunk);
      const int rem = u - ii * nb * nchunk;
      const int b = rem / nchunk, rc = rem - (rem / nchunk) * nchunk;
      const IItem item = p.items[it0 + ii];
      const int b0 = b * INNER_NC;
      const int nbat = min(INNER_NC, nact - b0);
      const int i0 = rc * w / nchunk, rows = (rc + 1) * w / nchunk - i0;
      const int Gc = blockDim.x / rows;
      if (item.cell >= 0) {
        // ---- stage slot panels in smem: pan[s][qq][j]
        for (int e = tid; e < 4 * INNER_NC * w; e += blockDim.x) {
          const int s = e / (INNER_NC * w);
          const int r2 = e - s * INNER_NC * w;
          const int qq = r2 / w, j = r2 - qq * w;
          double2 v = czero();
          if (qq < nbat && item.pan[s][0].vec >= 0) {
            const int r = act[b0 + qq];
            v = ld_cg(vecp(p, job, r, vmap[item.pan[s][0].vec]) + item.pan[s][0].seg * w + j);
            if (item.pan[s][1].vec >= 0)
              v = cadd(v, ld_cg(vecp(p, job, r, vmap[item.pan[s][1].vec]) + item.pan[s][1].seg * w + j));
          }
          pan[(s * INNER_NC + qq) * w + j] = v;
        }
        __syncthreads();
        if (tid < Gc * rows) {
          const int mi = tid % rows, mg = tid / rows;
          double2 acc[INNER_NC];
#pragma unroll
          for (int qq = 0; qq < INNER_NC; ++qq) acc[qq] = czero();
          const CellInfo& cell = p.cells[layer * p.Lc + item.cell];
          for (int s = 0; s < 4; ++s) {
            if (item.pan[s][0].vec < 0) continue;
            const double2* Gb = p.green + cell.green_off + (size_t)(item.row * 4 + s) * w * w + i0 + mi;
            const double2* ps = pan + (size_t)s * INNER_NC * w;
            for (int j = mg; j < w; j += Gc) {
              const double2 a = __ldg(Gb + (size_t)j * w);
#pragma unroll
              for (int qq = 0; qq < INNER_NC; ++qq) cfma(acc[qq], a, ps[qq * w + j]);
            }
          }
#pragma unroll
          for (int qq = 0; qq < INNER_NC; ++qq) red[(mg * rows + mi) * INNER_NC + qq] = acc[qq];
        }
        __syncthreads();
      }
      // ---- combine: out = y + add - (sub0 + sub1)
      for (int e = tid; e < nbat * rows; e += blockDim.x) {
        const int qq = e / rows, i = i0 + (e - qq * rows);
        const int r = act[b0 + qq];
        double2 y = czero();
        if (item.cell >= 0) {
          const int li = i - i0;
          y = red[li * INNER_NC + qq];
          for (int g = 1; g < Gc; ++g) y = cadd(y, red[(g * rows + li) * INNER_NC + qq]);
        }
        if (item.add.vec >= 0) y = cadd(y, ld_cg(vecp(p, job, r, vmap[item.add.vec]) + item.add.seg * w + i));
        if (item.sub[0].vec >= 0) {
          double2 sb = ld_cg(vecp(p, job, r, vmap[item.sub[0].vec]) + item.sub[0].seg * w + i);
          if (item.sub[1].vec >= 0)
            sb = cadd(sb, ld_cg(vecp(p, job, r, vmap[item.sub[1].vec]) + item.sub[1].seg * w + i));
          y = csub(y, sb);
        }
        vecp(p, job, r, vmap[item.dst.vec])[item.dst.seg * w + i] = y;
      }
      __syncthreads();
    }
    csync();
  }
}

// rebuild the (cluster-consistent) list of active instances from global state
__device__ __forceinline__ void rebuild_active(const InnerParams& p, int job, int* act, int* s_nact) {
  if (threadIdx.x == 0) {
    int na = 0;
    for (int r = 0; r < p.R; ++r)
      if (__ldcg(p.state + job * p.R + r) == 0) act[na++] = r;
    *s_nact = na;
  }
  __syncthreads();
}

__global__ void __cluster_dims__(INNER_CS, 1, 1) __launch_bounds__(PT_THREADS)
    inner_gmres_kernel(const InnerParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int CS = INNER_CS;
  const int q = (int)cg::this_cluster().block_rank();
  const int job = p.stage_jobs[blockIdx.x / CS];
  const int layer = p.jobs[job].layer;
  const int w = p.layers[layer].w;
  const int nIc = p.Lc - 1;
  const int n = 4 * nIc * w;
  const int tid = threadIdx.x;

  double2* pan = reinterpret_cast<double2*>(smem);
  double2* red = pan + 4 * INNER_NC * w;
  double* dred = reinterpret_cast<double*>(red + (size_t)PT_THREADS * INNER_NC);
  int* act = reinterpret_cast<int*>(dred + 64);
  __shared__ int s_nact, s_st;
  if (nIc == 0) return;
  const int VB = p.cap + 1, VY = p.cap + 2, VT = p.cap + 3, VA = p.cap + 4;
  const size_t hld = (size_t)p.cap + 1;
  auto Hp = [&](int r) { return p.hess + (size_t)(job * p.R + r) * p.hstride; };

  // ---- rhs_pol from the Newton tables (sie.py:230-242, negated); elements split over the cluster
  for (int r = 0; r < p.R; ++r) {
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
  if (tid < p.R) act[tid] = tid;
  if (tid == 0) s_nact = p.R;
  csync();

  // ---- b = pre(rhs), beta0 = ||b||, V_0 = b / beta0 (krylov.py:61-80)
  {
    const int vm[3] = {VB, VY, VA};
    run_program(p, job, layer, w, p.pre_ph, p.pre_nph, vm, act, s_nact, pan, red, q, CS);
  }
  for (int r = q; r < p.R; r += CS) {
    const double2* Y = vecp(p, job, r, VY);
    double ss = 0.0;
    for (int e = tid; e < n; e += blockDim.x) {
      const double2 y = ld_cg(Y + e);
      ss += y.x * y.x + y.y * y.y;
    }
    ss = block_sum(ss, dred);
    const double b0 = sqrt(ss);
    double2* V0 = vecp(p, job, r, 0);
    if (b0 != 0.0)
      for (int e = tid; e < n; e += blockDim.x) {
        const double2 y = ld_cg(Y + e);
        V0[e] = make_double2(y.x / b0, y.y / b0);
      }
    if (tid == 0) {
      double2* g = Hp(r) + hld * p.cap;
      g[0] = make_double2(b0, 0.0);
      p.beta0[job * p.R + r] = b0;
      p.state[job * p.R + r] = b0 == 0.0 ? 1 : 0;
      p.iters[job * p.R + r] = b0 == 0.0 ? 0 : -1;
    }
    __syncthreads();
  }
  csync();
  rebuild_active(p, job, act, &s_nact);

  for (int j = 0; j < p.max_iter && s_nact > 0; ++j) {
    const int nact = s_nact;
    if (j + 1 > p.cap) {  // basis capacity exhausted: the host retries with a larger capacity
      for (int a = 0; a < nact; ++a) {
        const int r = act[a];
        if (r % CS == q && tid == 0) {
          p.state[job * p.R + r] = 2;
          p.iters[job * p.R + r] = -1;
          atomicMax(p.err, 5);
        }
      }
      csync();
      rebuild_active(p, job, act, &s_nact);
      break;
    }
    {
      const int vm1[3] = {j, VT, VA};
      run_program(p, job, layer, w, p.op_ph, p.op_nph, vm1, act, nact, pan, red, q, CS);
      const int vm2[3] = {VT, j + 1, VA};
      run_program(p, job, layer, w, p.pre_ph, p.pre_nph, vm2, act, nact, pan, red, q, CS);
    }
    // ---- MGS Arnoldi + Givens for the instances this CTA owns (krylov.py:89-127)
    for (int a = 0; a < nact; ++a) {
      const int r = act[a];
      if (r % CS != q) continue;
      double2* W = vecp(p, job, r, j + 1);
      double2* H = Hp(r);
      double2* col = H + (size_t)j * hld;
      for (int i = 0; i <= j; ++i) {
        const double2* Vi = vecp(p, job, r, i);
        double sr = 0.0, si = 0.0;
        for (int e = tid; e < n; e += blockDim.x) {
          const double2 c = cconjmul(ld_cg(Vi + e), ld_cg(W + e));
          sr += c.x;
          si += c.y;
        }
        sr = block_sum(sr, dred);
        si = block_sum(si, dred);
        const double2 h = make_double2(sr, si);
        if (tid == 0) col[i] = h;
        for (int e = tid; e < n; e += blockDim.x) W[e] = csub(ld_cg(W + e), cmul(h, ld_cg(Vi + e)));
        __syncthreads();
      }
      double ss = 0.0;
      for (int e = tid; e < n; e += blockDim.x) {
        const double2 x = W[e];
        ss += x.x * x.x + x.y * x.y;
      }
      ss = block_sum(ss, dred);
      const double hn = sqrt(ss);
      if (tid == 0) {
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
      if (s_st == 0)  // V_{j+1} = w / hn (krylov.py:125)
        for (int e = tid; e < n; e += blockDim.x) {
          const double2 x = W[e];
          W[e] = make_double2(x.x / hn, x.y / hn);
        }
      __syncthreads();
    }
    csync();
    rebuild_active(p, job, act, &s_nact);
  }

  // ---- x = V_k y, traces = down + up (nested.py:153), owner CTA per instance
  double2* yv = pan;  // reuse smem: y[cap]
  for (int r = q; r < p.R; r += CS) {
    const int k = p.iters[job * p.R + r];
    if (tid == 0 && k > 0) {
      const double2* H = Hp(r);
      const double2* g = H + hld * p.cap;
      for (int i = k - 1; i >= 0; --i) {
        double2 s = czero();
        for (int l = i + 1; l < k; ++l) cfma(s, H[(size_t)l * hld + i], yv[l]);
        const double2 num = csub(g[i], s);
        const double2 den = H[(size_t)i * hld + i];
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
}

size_t inner_smem_bytes(int wmax, int R) {
  const int w = wmax < 8 ? 8 : wmax;
  return (size_t)4 * INNER_NC * w * 16 + (size_t)PT_THREADS * INNER_NC * 16 + 64 * 8 + (size_t)R * 4 + 64;
}

cudaError_t inner_launch(const InnerParams& p, int njobs, cudaStream_t st) {
  if (njobs == 0 || p.Lc < 2) return cudaSuccess;
  const size_t sm = inner_smem_bytes(p.wmax, p.R);
  cudaFuncSetAttribute(inner_gmres_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  inner_gmres_kernel<<<njobs * INNER_CS, PT_THREADS, sm, st>>>(p);
  return cudaGetLastError();
}
