// K1: batched cell solves H_c X = B by block-tridiagonal substitution with
// precomputed dense Schur inverses (replaces SuperLU.solve, subdomain.py:214-221).
//
//   forward   z_k = S_k^{-1} (b_k - l_k z_{k-1})          k = 0 .. wz_c-1
//   backward  x_k = z_k - u_k S_k^{-1} x_{k+1}            k = wz_c-2 .. 0
//
// One CTA per task = (cell, up to NC columns).  A column is one (layer-solve job,
// RHS) pair.  The right-hand side b_k is generated on the fly in the prologue of
// every step from the job description (equivalent interface sources at the four
// cut rows, the split volume source, and -- on the reconstruction pass -- the
// cell trace sources), so no layer volume is ever materialised.  The epilogue
// writes only what the caller consumes: the four Newton rows of each cell, the
// sampled layer rows, or the full stitched volume.
//
// S_k^{-1} does not depend on data, so it is streamed through an NS-slot shared
// memory ring by 1-D bulk async copies (cp.async.bulk, SASS UBLKCP) issued
// NS chunks ahead of the consumer; every byte of the factor is read exactly once
// per pass from HBM/L2.
#include "pt_device.cuh"

#include "pt_launch.cuh"


struct ColInfo {
  int jid, r, panmask, vol;  // vol: 0 none, 1 split slab of the global f, 2 full layer slab
};

template <int NC>
__global__ void __launch_bounds__(PT_THREADS) k1_cell_solve(const K1Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const K1Task task = p.tasks[blockIdx.x];
  const CellInfo cell = p.cells[task.cell];
  const LayerInfo lay = p.layers[cell.layer];
  const int w = cell.w, wzc = cell.wzc;
  const int tid = threadIdx.x;
  const int G = blockDim.x / w;
  const int nIc = p.Lc - 1;

  // ---- shared memory carve-up
  unsigned char* ring = smem;
  double2* va = reinterpret_cast<double2*>(ring + (size_t)p.ns * p.slot_bytes);
  double2* vb = va + w * NC;
  double2* red = vb + w * NC;
  ColInfo* cols = reinterpret_cast<ColInfo*>(red + (size_t)G * w * NC);
  uint64_t* full = reinterpret_cast<uint64_t*>(cols + NC + (NC & 1));

  const int jc = max(1, min(w, p.slot_bytes / (w * 16)));
  const int nch = (w + jc - 1) / jc;
  const int nsteps = 2 * wzc - 1;
  const int total = nsteps * nch;
  const double2* S = p.sinv + cell.sinv_off;

  auto issue = [&](int s) {
    const int st = s / nch, ch = s - st * nch;
    const int kmat = st < wzc ? st : 2 * wzc - 2 - st;
    const int c0 = ch * jc;
    const int cw = min(jc, w - c0);
    const uint32_t bytes = (uint32_t)cw * w * 16u;
    uint64_t* bar = &full[s % p.ns];
    mbar_expect_tx(bar, bytes);
    bulk_g2s(ring + (size_t)(s % p.ns) * p.slot_bytes, S + (size_t)kmat * w * w + (size_t)c0 * w, bytes, bar);
  };

  if (tid < NC) {
    ColInfo ci{-1, 0, 0, 0};
    if (tid < task.nq) {
      const int q = task.q0 + tid;
      if (p.pass == 2) {
        ci.jid = 0;
        ci.r = q;
      } else {
        ci.jid = p.ljobs[task.jb + q / p.R];
        ci.r = q % p.R;
        const OJob& jb = p.jobs[ci.jid];
        int m = 0;
        for (int s = 0; s < 4; ++s)
          if (jb.pan[s][0].vec >= 0) m |= 1 << s;
        ci.panmask = m;
        ci.vol = jb.vol ? (jb.vfull ? 2 : 1) : 0;
      }
    }
    cols[tid] = ci;
  }
  if (tid == 0) {
    for (int s = 0; s < p.ns; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < min(p.ns, total); ++s) issue(s);

  const bool active = tid < G * w;
  const int mi = tid % w, mg = tid / w;
  double2 acc[NC];
  int s = 0;

  // one matvec y = S_kmat^{-1} vin, reduced into red-sum per (i,q); returns via red buffer
  auto matvec = [&](const double2* vin) {
#pragma unroll
    for (int q = 0; q < NC; ++q) acc[q] = czero();
    for (int ch = 0; ch < nch; ++ch, ++s) {
      mbar_wait(&full[s % p.ns], (uint32_t)((s / p.ns) & 1));
      const double2* slot = reinterpret_cast<const double2*>(ring + (size_t)(s % p.ns) * p.slot_bytes);
      const int c0 = ch * jc;
      const int cw = min(jc, w - c0);
      if (active) {
        for (int jj = mg; jj < cw; jj += G) {
          const double2 a = slot[jj * w + mi];
          const double2* tv = vin + (c0 + jj) * NC;
#pragma unroll
          for (int q = 0; q < NC; ++q) cfma(acc[q], a, tv[q]);
        }
      }
      __syncthreads();
      if (tid == 0 && s + p.ns < total) issue(s + p.ns);
    }
    if (active) {
#pragma unroll
      for (int q = 0; q < NC; ++q) red[(mg * w + mi) * NC + q] = acc[q];
    }
    __syncthreads();
  };
  auto reduced = [&](int i, int q) {
    double2 y = red[i * NC + q];
    for (int g = 1; g < G; ++g) y = cadd(y, red[(g * w + i) * NC + q]);
    return y;
  };

  // right-hand side element b_k[j] of column q
  auto rhs = [&](int k, int j, int q) -> double2 {
    const ColInfo ci = cols[q];
    if (ci.jid < 0) return czero();
    if (p.pass == 2) return p.bd[((size_t)ci.r * wzc + k) * w + j];
    double2 inner = czero();
    if (k >= cell.lo && k < cell.hi) {
      const int X = cell.off + k;
#pragma unroll
      for (int sl = 0; sl < 4; ++sl)
        if ((ci.panmask >> sl & 1) && j == lay.prow[sl])
          inner = cadd(inner, cmul(lay.coef[sl], p.P[((size_t)(ci.jid * 4 + sl) * p.R + ci.r) * p.wx + X]));
      if (ci.vol == 1 && j >= lay.lo && j < lay.hi)
        inner = cadd(inner, p.f[ci.r * p.f_stride + (size_t)(lay.off + j) * p.wx + X]);
      else if (ci.vol == 2)
        inner = cadd(inner, p.f[ci.r * p.f_stride + (size_t)j * p.wx + X]);
    }
    if (p.pass == 1) {
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        const bool has = sl < 2 ? cell.has_top : cell.has_bot;
        if (has && k == cell.krow[sl]) {
          const int I = sl < 2 ? cell.cell - 1 : cell.cell;
          const double2 t =
              p.tr[((((size_t)ci.jid * p.R + ci.r) * nIc + I) * 2 + (sl & 1)) * p.wmax + j];
          return cadd(cmul(cell.coef[sl], t), inner);
        }
      }
    }
    return inner;
  };

  // epilogue of backward step k: x_k lives in vx ([w][NC])
  auto emit = [&](int k, const double2* vx) {
    for (int e = tid; e < w * NC; e += blockDim.x) {
      const int i = e / NC, q = e - (e / NC) * NC;
      const ColInfo ci = cols[q];
      if (ci.jid < 0) continue;
      const double2 x = vx[e];
      if (p.pass == 2) {
        p.xd[((size_t)ci.r * wzc + k) * w + i] = x;
      } else if (p.pass == 0) {
#pragma unroll
        for (int idx = 0; idx < 4; ++idx) {
          const bool need = idx < 2 ? cell.has_top : cell.has_bot;
          if (need && k == cell.srow[idx])
            p.tables[((((size_t)ci.jid * p.Lc + cell.cell) * 4 + idx) * p.R + ci.r) * p.wmax + i] = x;
        }
      } else if (k >= cell.lo && k < cell.hi) {
        const int X = cell.off + k;
        const OJob& jb = p.jobs[ci.jid];
        if (jb.nout < 0) {
          if (jb.vfull)
            p.u[ci.r * p.u_stride + (size_t)i * p.wx + X] = x;
          else if (i >= lay.lo && i < lay.hi)
            p.u[ci.r * p.u_stride + (size_t)(lay.off + i) * p.wx + X] = x;
        } else {
          for (int o = 0; o < jb.nout; ++o)
            if (i == jb.orow[o] + p.npml - 1) p.smp[((size_t)(ci.jid * 4 + o) * p.R + ci.r) * p.wx + X] = x;
        }
      }
    }
  };

  double2* Z = p.Z + task.zoff;
  // ---------------- forward sweep
  double2* vin = va;
  double2* vz = vb;  // z_{k-1}
  for (int k = 0; k < wzc; ++k) {
    const double2 lk = p.lz[cell.lz_off + k];
    for (int e = tid; e < w * NC; e += blockDim.x) {
      const int j = e / NC, q = e - (e / NC) * NC;
      double2 b = rhs(k, j, q);
      if (k > 0) b = csub(b, cmul(lk, vz[e]));
      vin[e] = b;
    }
    __syncthreads();
    matvec(vin);
    for (int e = tid; e < w * NC; e += blockDim.x) {
      const int i = e / NC, q = e - (e / NC) * NC;
      const double2 y = reduced(i, q);
      vz[e] = y;
      Z[(size_t)k * w * NC + e] = y;
    }
    __syncthreads();
  }
  // ---------------- backward sweep: vz holds z_{wzc-1} = x_{wzc-1}
  emit(wzc - 1, vz);
  double2* vx = vz;
  double2* vo = va;
  for (int k = wzc - 2; k >= 0; --k) {
    __syncthreads();
    matvec(vx);
    const double2 uk = p.uz[cell.lz_off + k];
    for (int e = tid; e < w * NC; e += blockDim.x) {
      const int i = e / NC, q = e - (e / NC) * NC;
      const double2 y = reduced(i, q);
      vo[e] = csub(Z[(size_t)k * w * NC + e], cmul(uk, y));
    }
    __syncthreads();
    emit(k, vo);
    double2* t = vx;
    vx = vo;
    vo = t;
  }
}

size_t k1_smem_bytes(int wmax, int nc, int slot_bytes, int ns) {
  // ring + two [w][NC] vectors + the [G][w][NC] reduction buffer (G*w <= 256) + column info + barriers
  return (size_t)ns * slot_bytes + (size_t)(2 * wmax + PT_THREADS) * nc * 16 + (size_t)(nc + 2) * 16 + 16 +
         (size_t)ns * 8;
}

cudaError_t k1_launch(const K1Params& p, int ntasks, int nc, int wmax, cudaStream_t st) {
  if (ntasks == 0) return cudaSuccess;
  const size_t smax = k1_smem_bytes(wmax, nc, p.slot_bytes, p.ns);
  switch (nc) {
#define PT_K1_CASE(N)                                                                                \
  case N:                                                                                            \
    cudaFuncSetAttribute(k1_cell_solve<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax); \
    k1_cell_solve<N><<<ntasks, PT_THREADS, smax, st>>>(p);                                           \
    break;
    PT_K1_CASE(1)
    PT_K1_CASE(2)
    PT_K1_CASE(4)
    PT_K1_CASE(8)
#undef PT_K1_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
