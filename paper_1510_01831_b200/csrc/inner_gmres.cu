// Inner polarized-traces GMRES (replaces _InnerPT.solve_traces, nested.py:134-153).
//
// One CTA per layer-solve job; the job's R right-hand-side instances advance
// in lockstep and are frozen individually when they converge, so every
// instance runs exactly the Krylov process of krylov.gmres (krylov.py:53-135):
// same operator (inner apply_M_polarized on the dense Green blocks,
// sie.py:203-228 / nested.py:113-122), same left GS preconditioner
// (sie.py:272-326), MGS Arnoldi with vdot, complex Givens, stop when
// |g_{j+1}|/beta0 <= inner_ktol, x = V_k y.  The data-dependent iteration
// count never leaves the device.
//
// The operator and preconditioner are executed from "item programs" built on
// the host: each item is one sampled panel = sum_slot G[cell][row][slot] @
// panel_slot + add - (sub0 + sub1), which is exactly the arithmetic of the
// reference's TraceSystem methods; items of one phase are independent.
#include "pt_device.cuh"


#include "pt_launch.cuh"


__device__ __forceinline__ double2* vecp(const InnerParams& p, int job, int r, int v) {
  return p.scratch + (size_t)(job * p.R + r) * p.inst_stride + (size_t)v * p.nmax;
}

// Execute one program (list of phases) for the active instances.
// vmap: program vec ids {0:IN,1:OUT,2:AUX} -> scratch vector index.
__device__ void run_program(const InnerParams& p, int job, int layer, int w, const int* ph, int nph,
                            const int vmap[3], const int* act, int nact, double2* pan, double2* red) {
  const int tid = threadIdx.x;
  const int G = blockDim.x / w;
  const bool mact = tid < G * w;
  const int mi = tid % w, mg = tid / w;
  const int nseg_w = w;
  for (int phz = 0; phz < nph; ++phz) {
    for (int it = ph[phz]; it < ph[phz + 1]; ++it) {
      const IItem item = p.items[it];
      for (int b0 = 0; b0 < nact; b0 += INNER_NC) {
        const int nb = min(INNER_NC, nact - b0);
        // ---- stage slot panels in smem: pan[s][q][j]
        if (item.cell >= 0) {
          for (int e = tid; e < 4 * INNER_NC * w; e += blockDim.x) {
            const int s = e / (INNER_NC * w);
            const int rem = e - s * INNER_NC * w;
            const int q = rem / w, j = rem - q * w;
            double2 v = czero();
            if (q < nb && item.pan[s][0].vec >= 0) {
              const int r = act[b0 + q];
              v = ld_cg(vecp(p, job, r, vmap[item.pan[s][0].vec]) + item.pan[s][0].seg * nseg_w + j);
              if (item.pan[s][1].vec >= 0)
                v = cadd(v, ld_cg(vecp(p, job, r, vmap[item.pan[s][1].vec]) + item.pan[s][1].seg * nseg_w + j));
            }
            pan[(s * INNER_NC + q) * w + j] = v;
          }
          __syncthreads();
          double2 acc[INNER_NC];
#pragma unroll
          for (int q = 0; q < INNER_NC; ++q) acc[q] = czero();
          if (mact) {
            const CellInfo& cell = p.cells[layer * p.Lc + item.cell];
            for (int s = 0; s < 4; ++s) {
              if (item.pan[s][0].vec < 0) continue;
              const double2* Gb = p.green + cell.green_off + (size_t)(item.row * 4 + s) * w * w;
              const double2* ps = pan + (size_t)s * INNER_NC * w;
              for (int j = mg; j < w; j += G) {
                const double2 a = __ldg(Gb + (size_t)j * w + mi);
#pragma unroll
                for (int q = 0; q < INNER_NC; ++q) cfma(acc[q], a, ps[q * w + j]);
              }
            }
#pragma unroll
            for (int q = 0; q < INNER_NC; ++q) red[(mg * w + mi) * INNER_NC + q] = acc[q];
          }
          __syncthreads();
        }
        // ---- combine: out = y + add - (sub0 + sub1)
        for (int e = tid; e < nb * w; e += blockDim.x) {
          const int q = e / w, i = e - q * w;
          const int r = act[b0 + q];
          double2 y = czero();
          if (item.cell >= 0) {
            y = red[i * INNER_NC + q];
            for (int g = 1; g < G; ++g) y = cadd(y, red[(g * w + i) * INNER_NC + q]);
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
    }
  }
}

__global__ void __launch_bounds__(PT_THREADS) inner_gmres_kernel(const InnerParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int job = p.stage_jobs[blockIdx.x];
  const int layer = p.jobs[job].layer;
  const int w = p.layers[layer].w;
  const int nIc = p.Lc - 1;
  const int n = 4 * nIc * w;
  const int tid = threadIdx.x;
  const int G = blockDim.x / w;

  double2* pan = reinterpret_cast<double2*>(smem);
  double2* red = pan + 4 * INNER_NC * w;
  double* dred = reinterpret_cast<double*>(red + (size_t)G * w * INNER_NC);
  int* act = reinterpret_cast<int*>(dred + 64);
  int* state = act + p.R;  // per instance: 0 active, 1 done, 2 error
  double* beta0 = reinterpret_cast<double*>(state + p.R);  // act is 8-byte aligned, 2R ints
  __shared__ int s_nact;

  if (nIc == 0) return;
  const int VB = p.cap + 1, VY = p.cap + 2, VT = p.cap + 3, VA = p.cap + 4;

  // ---- rhs_pol from the Newton tables (sie.py:230-242, negated)
  for (int r = 0; r < p.R; ++r) {
    double2* B = vecp(p, job, r, VB);
    for (int e = tid; e < n; e += blockDim.x) {
      const int seg = e / w, j = e - seg * w;
      const int half = seg / (2 * nIc);  // 0 down, 1 up
      const int I = (seg % (2 * nIc)) / 2, s = seg & 1;
      const int c = half == 0 ? I : I + 1;
      const int idx = half == 0 ? 2 + s : s;  // down: rn, rnp of cell I; up: r0, r1 of cell I+1
      const double2 t = p.tables[((((size_t)job * p.Lc + c) * 4 + idx) * p.R + r) * p.wmax + j];
      B[e] = make_double2(-t.x, -t.y);
    }
  }
  if (tid < p.R) {
    act[tid] = tid;
    state[tid] = 0;
  }
  if (tid == 0) s_nact = p.R;
  __syncthreads();

  // ---- b = pre(rhs)
  {
    const int vm[3] = {VB, VY, VA};
    run_program(p, job, layer, w, p.pre_ph, p.pre_nph, vm, act, s_nact, pan, red);
  }
  for (int r = 0; r < p.R; ++r) {
    const double2* Y = vecp(p, job, r, VY);
    double ss = 0.0;
    for (int e = tid; e < n; e += blockDim.x) ss += Y[e].x * Y[e].x + Y[e].y * Y[e].y;
    ss = block_sum(ss, dred);
    const double b0 = sqrt(ss);
    if (tid == 0) beta0[r] = b0;
    double2* V0 = vecp(p, job, r, 0);
    if (b0 != 0.0) {
      for (int e = tid; e < n; e += blockDim.x) V0[e] = make_double2(Y[e].x / b0, Y[e].y / b0);
    }
    __syncthreads();
  }
  if (tid == 0) {
    int na = 0;
    for (int r = 0; r < p.R; ++r) {
      double2* hg = p.hess + (size_t)(job * p.R + r) * p.hstride + (size_t)(p.cap + 1) * p.cap;
      hg[0] = make_double2(beta0[r], 0.0);
      if (beta0[r] == 0.0) {
        state[r] = 1;
        p.iters[job * p.R + r] = 0;
      } else {
        act[na++] = r;
      }
    }
    s_nact = na;
  }
  __syncthreads();

  for (int j = 0; j < p.max_iter && s_nact > 0; ++j) {
    if (j + 1 > p.cap) {
      if (tid == 0) {
        for (int a = 0; a < s_nact; ++a) {
          state[act[a]] = 2;
          p.iters[job * p.R + act[a]] = -1;
        }
        atomicMax(p.err, 5);
        s_nact = 0;
      }
      __syncthreads();
      break;
    }
    const int nact = s_nact;
    {
      const int vm1[3] = {j, VT, VA};
      run_program(p, job, layer, w, p.op_ph, p.op_nph, vm1, act, nact, pan, red);
      const int vm2[3] = {VT, j + 1, VA};
      run_program(p, job, layer, w, p.pre_ph, p.pre_nph, vm2, act, nact, pan, red);
    }
    // ---- MGS Arnoldi per active instance (krylov.py:89-94)
    for (int a = 0; a < nact; ++a) {
      const int r = act[a];
      double2* W = vecp(p, job, r, j + 1);
      double2* H = p.hess + (size_t)(job * p.R + r) * p.hstride;
      for (int i = 0; i <= j; ++i) {
        const double2* Vi = vecp(p, job, r, i);
        double sr = 0.0, si = 0.0;
        for (int e = tid; e < n; e += blockDim.x) {
          const double2 c = cconjmul(Vi[e], W[e]);
          sr += c.x;
          si += c.y;
        }
        sr = block_sum(sr, dred);
        si = block_sum(si, dred);
        const double2 h = make_double2(sr, si);
        if (tid == 0) H[(size_t)j * (p.cap + 1) + i] = h;
        for (int e = tid; e < n; e += blockDim.x) W[e] = csub(W[e], cmul(h, Vi[e]));
        __syncthreads();
      }
      double ss = 0.0;
      for (int e = tid; e < n; e += blockDim.x) ss += W[e].x * W[e].x + W[e].y * W[e].y;
      ss = block_sum(ss, dred);
      if (tid == 0) H[(size_t)j * (p.cap + 1) + j + 1] = make_double2(sqrt(ss), 0.0);
      __syncthreads();
    }
    // ---- Givens + convergence per instance (krylov.py:95-127), one thread each
    if (tid < nact) {
      const int r = act[tid];
      double2* H = p.hess + (size_t)(job * p.R + r) * p.hstride;
      double2* g = H + (size_t)(p.cap + 1) * p.cap;
      double2* cs = g + (p.cap + 1);
      double2* sn = cs + p.cap;
      double2* col = H + (size_t)j * (p.cap + 1);
      const double hn = col[j + 1].x;
      for (int i = 0; i < j; ++i) {
        const double2 t = cadd(cmul(cs[i], col[i]), cmul(sn[i], col[i + 1]));
        const double2 nsc = make_double2(-sn[i].x, sn[i].y);   // -conj(sn)
        const double2 csc = make_double2(cs[i].x, -cs[i].y);   // conj(cs)
        col[i + 1] = cadd(cmul(nsc, col[i]), cmul(csc, col[i + 1]));
        col[i] = t;
      }
      const double a = hypot(col[j].x, col[j].y);
      const double d = sqrt(a * a + hn * hn);
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
        const double res = hypot(g[j + 1].x, g[j + 1].y) / beta0[r];
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
      state[r] = st;
      if (st != 0) p.iters[job * p.R + r] = st == 1 ? j + 1 : -1;
    }
    __syncthreads();
    // ---- V_{j+1} = w / hn for continuing instances
    for (int a = 0; a < nact; ++a) {
      const int r = act[a];
      if (state[r] != 0) continue;
      double2* W = vecp(p, job, r, j + 1);
      const double2* H = p.hess + (size_t)(job * p.R + r) * p.hstride;
      const double hn = H[(size_t)j * (p.cap + 1) + j + 1].x;
      for (int e = tid; e < n; e += blockDim.x) W[e] = make_double2(W[e].x / hn, W[e].y / hn);
    }
    __syncthreads();
    if (tid == 0) {
      int na = 0;
      for (int a = 0; a < nact; ++a)
        if (state[act[a]] == 0) act[na++] = act[a];
      s_nact = na;
    }
    __syncthreads();
  }

  // ---- x = V_k y, traces = down + up (nested.py:153)
  for (int r = 0; r < p.R; ++r) {
    const int k = p.iters[job * p.R + r];
    double2* yv = reinterpret_cast<double2*>(pan);  // reuse smem: y[cap]
    if (tid == 0 && k > 0) {
      const double2* H = p.hess + (size_t)(job * p.R + r) * p.hstride;
      const double2* g = H + (size_t)(p.cap + 1) * p.cap;
      for (int i = k - 1; i >= 0; --i) {
        double2 s = czero();
        for (int l = i + 1; l < k; ++l) cfma(s, H[(size_t)l * (p.cap + 1) + i], yv[l]);
        const double2 num = csub(g[i], s);
        const double2 den = H[(size_t)i * (p.cap + 1) + i];
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
        cfma(xd, Vi[e], yv[i]);
        cfma(xu, Vi[half + e], yv[i]);
      }
      const int seg = e / w, j = e - seg * w;
      out[(size_t)seg * p.wmax + j] = cadd(xd, xu);
    }
    __syncthreads();
  }
  // ---- accounting: TouchCounter.total equivalent (nested.py:54-73)
  if (tid < p.R) {
    const int its = p.iters[job * p.R + tid];
    if (its >= 0) {
      atomicAdd(&p.hist[min(its, PT_HIST - 1)], 1);
      atomicAdd(&p.counters[0], (unsigned long long)its);
      const unsigned long long t =
          ((unsigned long long)(its + 1) * p.pre_blocks + (unsigned long long)its * p.op_blocks) * w * w;
      atomicAdd(&p.counters[1], t);
      atomicAdd(&p.counters[2], 1ULL);
    }
  }
}

size_t inner_smem_bytes(int wmax, int R) {
  const int w = wmax < 8 ? 8 : wmax;
  return (size_t)4 * INNER_NC * w * 16 + (size_t)(PT_THREADS + 2 * w) * INNER_NC * 16 + 64 * 8 +
         (size_t)(2 * R + 2) * 4 + (size_t)R * 8 + 64;
}

cudaError_t inner_launch(const InnerParams& p, int njobs, cudaStream_t st) {
  if (njobs == 0 || p.Lc < 2) return cudaSuccess;
  const size_t sm = inner_smem_bytes(p.wmax, p.R);
  cudaFuncSetAttribute(inner_gmres_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  inner_gmres_kernel<<<njobs, PT_THREADS, sm, st>>>(p);
  return cudaGetLastError();
}
