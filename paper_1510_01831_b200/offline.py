"""Offline stage: per-cell Schur factors and interface Green blocks.

Everything here runs once per (model, frequency, partition) and is uploaded to
the device by ``pt_create``.  It replaces the reference's offline objects

* ``LayerWorkspace.__init__ -> spla.splu`` for every cell
  (``subdomain.py:202-212``, built by ``NestedLayerSolver.__init__``,
  ``nested.py:293-302``), and
* ``GreenBlockSet.build`` (``green.py:103-129``, ``nested.py:303-307``),

with the factorization the B200 online stage consumes:

**Cell operator.**  After the x<->z swap (``nested.py:45-47, 294-296``) a cell
of layer l has ``wz_c = nx_c + 2 npml`` block rows (original x columns) of
width ``w = n_l + 2 npml`` (original layer depth).  Its 5-point operator is
block tridiagonal (``discretization.py:251``)::

    H_c = tridiag(l_k I, D_k, u_k I),
    D_k = T_w + diag(tz_k - omega^2 m_k),   T_w tridiagonal (PML across w),

with scalar off-diagonal blocks ``l_k = T_z[k, k-1]``, ``u_k = T_z[k, k+1]``.

**Schur factors.**  ``S_0 = D_0``, ``S_k = D_k - l_k u_{k-1} S_{k-1}^{-1}``;
the dense inverses ``S_k^{-1}`` are stored.  A cell solve is then
``z_k = S_k^{-1}(b_k - l_k z_{k-1})`` forward and
``x_k = z_k - u_k S_k^{-1} x_{k+1}`` backward (kernel K1).

**Green blocks.**  ``G[(j, slot)] = coef_slot * (H_c^{-1})[row(j), row(slot)]``
for ``j in {0, 1, n, n+1}`` and the four slot sources of ``green.py:370-377``
(``v0: -l at row 1``, ``v1: +u at row 0``, ``vn: +l at row n+1``,
``vnp: -u at row n``).

All blocks are emitted COLUMN-MAJOR (element (i, j) at ``j*w + i``), the
layout K1 and the inner kernels read.  Computation uses torch so that the
same code runs on the CPU (tests) or batched on the GPU (large configs).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .discretization import axis_tridiag

__all__ = ["CellFactors", "LayerFactors", "Factors", "build_factors", "cut_coefs", "residual_from_operator"]

ROWS = ("r0", "r1", "rn", "rnp")  # sampled rows j = 0, 1, n, n+1
SLOTS = ("v0", "v1", "vn", "vnp")


def cut_coefs(lower, upper, npml, n):
    """Slot-source coefficients and positions of one slab.

    For a slab with ``n`` interior rows along its stacking axis whose 1-D
    operator has sub/super diagonals ``lower``/``upper``, ``src_top`` /
    ``src_bot`` (``subdomain.py:157-182``) place

    * v0 : ``-H_{1,0}``    at row(1)   -> ``-lower[row(1)]``
    * v1 : ``+H_{0,1}``    at row(0)   -> ``+upper[row(0)]``
    * vn : ``+H_{n+1,n}``  at row(n+1) -> ``+lower[row(n+1)]``
    * vnp: ``-H_{n,n+1}``  at row(n)   -> ``-upper[row(n)]``

    Returns ``(coefs[4] complex, rows[4] int)`` in slot order.
    """
    r = lambda k: k + npml - 1  # noqa: E731  (subdomain.py:133-138)
    rows = np.array([r(1), r(0), r(n + 1), r(n)], dtype=np.int64)
    coefs = np.array(
        [-lower[r(1)], upper[r(0)], lower[r(n + 1)], -upper[r(n)]], dtype=np.complex128
    )
    return coefs, rows


@dataclass
class CellFactors:
    layer: int
    cell: int
    w: int
    wzc: int
    nxc: int
    off: int
    sinv: torch.Tensor  # (wzc, w, w) complex128 twisted factors (see _twisted_inverses), column-major blocks
    lz: np.ndarray  # (wzc,) block-row couplings l_k
    uz: np.ndarray  # (wzc,) u_k
    green: torch.Tensor  # (4 rows, 4 slots, w, w) column-major blocks
    coefs: np.ndarray  # (4,) cell-level slot coefficients
    krows: np.ndarray  # (4,) cell block rows of the slot sources
    # (wzc, 4 layer trace rows, 4 slots, w): H_c^{-1} (coef_s E_{krow_s}) sampled at every block row
    # and at the layer trace rows 0, 1, n, n+1 -- the trace-source response of the sampled rows
    gsmp: torch.Tensor = None
    # (M, K) pass-0 operator for layer solves without a volume source: columns (slot s, kept block row k;
    # each slot block zero-padded to nk4 = roundup(nk, 4))
    # = lay.coef[s] E_{(k, prow_s)}, rows = the Newton-table block rows (4 x w, order r0 r1 rn rnp) then the
    # layer trace rows of every kept block row ((k, row) k-major, rows 0, 1, n, n+1); M padded to 8
    q0: torch.Tensor = None


@dataclass
class LayerFactors:
    index: int
    n: int
    off: int
    w: int
    coefs: np.ndarray  # (4,) layer-level slot coefficients
    prows: np.ndarray  # (4,) layer rows of the slot sources
    cells: list = field(default_factory=list)
    # (4, n, n) complex: the inner trace problem's dense preconditioner, pre o op, and the s-step operators
    # E pre, E^2 pre with E = pre o op - I (n = 4 (Lc-1) w)
    dense: torch.Tensor = None
    # (m, m) complex, m = 2 (Lc-1) w: inverse of the assembled cell-interface system of the direct
    # inner backend (backend="lu", nested.py:156-254)
    lu_inv: torch.Tensor = None


@dataclass
class Factors:
    nx: int
    nz: int
    h: float
    npml: int
    omega: float
    L: int
    Lc: int
    layers: list
    cell_extents: tuple
    cell_offsets: tuple
    tx: tuple  # global T_x diagonals (lower, main, upper), length wx
    tz: tuple  # global T_z diagonals, length wz
    m: np.ndarray  # (wz, wx) squared slowness
    # the reference's factored boundary pipeline (nested.py:355-486) is selected: same linear maps (this
    # path's pass-0 / sampled-response operators are M_f / direct / M_u), its touch accounting
    assembled_boundary: bool = False
    # optional (wz, wx) complex diagonal of a caller-supplied global operator (residual only)
    hdiag: np.ndarray = None

    @property
    def wx(self):
        return self.nx + 2 * self.npml

    @property
    def wz(self):
        return self.nz + 2 * self.npml

    def sinv_bytes(self):
        return sum(cf.sinv.numel() * 16 for lf in self.layers for cf in lf.cells)

    def green_bytes(self):
        return sum(cf.green.numel() * 16 for lf in self.layers for cf in lf.cells)


class _Timer:
    """Wall-clock totals of the offline phases (``PT_OFFLINE_TIMES=1`` prints them; device work is synchronised
    at every mark, so the switch serialises the stage)."""

    def __init__(self, device):
        import os

        self.on = bool(os.environ.get("PT_OFFLINE_TIMES"))
        self.device = device
        self.tot = {}
        self.t = None

    def mark(self, name=None):
        if not self.on:
            return
        import time

        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        now = time.perf_counter()
        if name is not None and self.t is not None:
            self.tot[name] = self.tot.get(name, 0.0) + now - self.t
        self.t = now

    def report(self):
        if self.on:
            import sys

            sys.stderr.write("offline times: " + ", ".join(f"{k} {v:.2f}s" for k, v in self.tot.items()) + "\n")


def _split(n, parts):
    base, rem = divmod(n, parts)
    return tuple(base + 1 if i < rem else base for i in range(parts))


def _schur_inverses(tw, diag, lz, uz, device):
    """Batched Schur recursion over cells of equal (w, wzc).

    ``tw``: (lower, main, upper) of T_w (length w, shared by the batch);
    ``diag``: (B, wzc, w) complex -- tz_k - omega^2 m_k per cell;
    ``lz``/``uz``: (wzc,) shared block couplings.  Returns (B, wzc, w, w)
    inverses in natural row-major orientation.
    """
    B, wzc, w = diag.shape
    lo, mn, up = (torch.as_tensor(a, dtype=torch.complex128, device=device) for a in tw)
    base = torch.diag(mn) + torch.diag(up[:-1], 1) + torch.diag(lo[1:], -1)
    out = torch.empty((B, wzc, w, w), dtype=torch.complex128, device=device)
    prev = None
    for k in range(wzc):
        S = base.expand(B, w, w).clone()
        S.diagonal(dim1=-2, dim2=-1).add_(diag[:, k, :])
        if k > 0:
            S -= (complex(lz[k]) * complex(uz[k - 1])) * prev
        prev = torch.linalg.inv(S)
        out[:, k] = prev
    return out


def _twisted_inverses(tw, diag, lz, uz, sinv_fwd, device):
    """Two-sided ("twisted") block factorization used by K1.

    Top blocks k < m keep the forward Schur inverses S_k^{-1}; bottom blocks
    k > m hold T_k^{-1} with T_{wz-1} = D_{wz-1}, T_k = D_k - u_k l_{k+1} T_{k+1}^{-1};
    the middle block holds M^{-1} with
    M = D_m - l_m u_{m-1} S_{m-1}^{-1} - u_m l_{m+1} T_{m+1}^{-1}, m = wz_c // 2.
    A solve is then two independent half-length chains that meet at block m.
    """
    B, wzc, w = diag.shape
    m = wzc // 2
    lo, mn, up = (torch.as_tensor(a, dtype=torch.complex128, device=device) for a in tw)
    base = torch.diag(mn) + torch.diag(up[:-1], 1) + torch.diag(lo[1:], -1)
    out = sinv_fwd.clone()
    prev = None
    for k in range(wzc - 1, m, -1):
        T = base.expand(B, w, w).clone()
        T.diagonal(dim1=-2, dim2=-1).add_(diag[:, k, :])
        if k < wzc - 1:
            T -= (complex(uz[k]) * complex(lz[k + 1])) * prev
        prev = torch.linalg.inv(T)
        out[:, k] = prev
    Mm = base.expand(B, w, w).clone()
    Mm.diagonal(dim1=-2, dim2=-1).add_(diag[:, m, :])
    if m > 0:
        Mm -= (complex(lz[m]) * complex(uz[m - 1])) * sinv_fwd[:, m - 1]
    if m < wzc - 1:
        Mm -= (complex(uz[m]) * complex(lz[m + 1])) * prev
    out[:, m] = torch.linalg.inv(Mm)
    return out


def _twisted_solve(tinv, lz, uz, rhs):
    """Solve with twisted factors (mirrors the K1 kernel's two half-chains)."""
    B, wzc, w, _ = tinv.shape
    m = wzc // 2
    z = torch.empty_like(rhs)
    prev = None
    for k in range(m):
        t = rhs[:, k] if k == 0 else rhs[:, k] - complex(lz[k]) * prev
        prev = tinv[:, k] @ t
        z[:, k] = prev
    zt = prev
    prev = None
    for k in range(wzc - 1, m, -1):
        t = rhs[:, k] if k == wzc - 1 else rhs[:, k] - complex(uz[k]) * prev
        prev = tinv[:, k] @ t
        z[:, k] = prev
    t = rhs[:, m]
    if m > 0:
        t = t - complex(lz[m]) * zt
    if m < wzc - 1:
        t = t - complex(uz[m]) * prev
    x = torch.empty_like(rhs)
    x[:, m] = tinv[:, m] @ t
    for k in range(m - 1, -1, -1):
        x[:, k] = z[:, k] - complex(uz[k]) * (tinv[:, k] @ x[:, k + 1])
    for k in range(m + 1, wzc):
        x[:, k] = z[:, k] - complex(lz[k]) * (tinv[:, k] @ x[:, k - 1])
    return x


def _block_solve(sinv, lz, uz, rhs):
    """Solve H_c X = RHS with stored Schur inverses (batched over cells).

    sinv: (B, wzc, w, w) row-major; rhs: (B, wzc, w, nrhs).  Mirrors K1.
    """
    B, wzc, w, _ = sinv.shape
    z = torch.empty_like(rhs)
    prev = None
    for k in range(wzc):
        t = rhs[:, k] if k == 0 else rhs[:, k] - complex(lz[k]) * prev
        prev = sinv[:, k] @ t
        z[:, k] = prev
    x = torch.empty_like(rhs)
    nxt = z[:, wzc - 1]
    x[:, wzc - 1] = nxt
    for k in range(wzc - 2, -1, -1):
        nxt = z[:, k] - complex(uz[k]) * (sinv[:, k] @ nxt)
        x[:, k] = nxt
    return x


def inner_dense_operators(lf):
    """Dense inner operators of one layer: ``(Pm, Bm)`` with ``Pm = pre`` and ``Bm = pre o op``.

    ``op`` is ``apply_M_polarized`` (``sie.py:203-228``) and ``pre`` the Gauss-Seidel
    preconditioner (``sweep_down``, ``upward_reflections``, ``sweep_up``: ``sie.py:272-329``)
    of the layer's inner trace problem, whose "slabs" are the cells and whose
    ``boundary_samples`` are the cell Green blocks (``nested.py:113-122``).  The trace
    vector is ``[down (nI, 2, w); up (nI, 2, w)]`` flattened.  Both maps are linear, so the
    inner GMRES (``nested.py:134-153``) can apply ``pre(op(v))`` as one dense product.
    Returns complex128 tensors of shape ``(n, n)``, ``n = 4 nI w``, or ``None`` for Lc == 1.
    """
    cells = lf.cells
    Lc = len(cells)
    nI = Lc - 1
    if nI == 0:
        return None
    w = lf.w
    n = 4 * nI * w
    dev = cells[0].green.device
    # row-major Green blocks G[c][row jr][slot s]: rows r0, r1, rn, rnp; slots v0, v1, vn, vnp
    G = [cf.green.transpose(-1, -2) for cf in cells]
    R0, R1, RN, RNP = 0, 1, 2, 3

    def bs(c, pans, rows):
        out = []
        for jr in rows:
            acc = None
            for s in range(4):
                if pans[s] is not None:
                    t = G[c][jr, s] @ pans[s]
                    acc = t if acc is None else acc + t
            out.append(acc)
        return out

    def unpack(X):
        return X[: 2 * nI * w].reshape(nI, 2, w, -1), X[2 * nI * w :].reshape(nI, 2, w, -1)

    def op(X):  # sie.py:203-228
        d, p = unpack(X)
        od = torch.zeros_like(d)
        ou = torch.zeros_like(p)
        for ell in range(1, Lc + 1):
            top, bot = ell >= 2, ell <= Lc - 1
            it, ib = ell - 2, ell - 1
            c = ell - 1
            if bot:
                v0 = d[ib - 1, 0] + p[ib - 1, 0] if top else None
                v1 = d[ib - 1, 1] + p[ib - 1, 1] if top else None
                wb = bs(c, [v0, v1, p[ib, 0], p[ib, 1]], (RN, RNP))
                od[ib, 0] = wb[0] - (d[ib, 0] + p[ib, 0])
                od[ib, 1] = wb[1] - d[ib, 1]
            if top:
                vn = p[ib, 0] + d[ib, 0] if bot else None
                vnp = p[ib, 1] + d[ib, 1] if bot else None
                wt = bs(c, [d[it, 0], d[it, 1], vn, vnp], (R0, R1))
                ou[it, 0] = wt[0] - p[it, 0]
                ou[it, 1] = wt[1] - (d[it, 1] + p[it, 1])
        return torch.cat([od.reshape(2 * nI * w, -1), ou.reshape(2 * nI * w, -1)])

    def pre(X):  # sie.py:272-329 (kind "gs")
        v, pv = unpack(X)
        yd = torch.zeros_like(v)
        yd[0] = -v[0]
        for i in range(2, nI + 1):  # sweep_down, slab i-1 = cell i-1, rows n, n+1
            wv = bs(i - 1, [yd[i - 2, 0], yd[i - 2, 1], None, None], (RN, RNP))
            yd[i - 1, 0] = wv[0] - v[i - 1, 0]
            yd[i - 1, 1] = wv[1] - v[i - 1, 1]
        refl = torch.zeros_like(v)
        for i in range(1, nI + 1):  # upward_reflections, slab i = cell i, rows 0, 1
            b0 = yd[i, 0] if i <= nI - 1 else None
            b1 = yd[i, 1] if i <= nI - 1 else None
            wv = bs(i, [yd[i - 1, 0], yd[i - 1, 1], b0, b1], (R0, R1))
            refl[i - 1, 0] = wv[0]
            refl[i - 1, 1] = wv[1] - yd[i - 1, 1]
        sv = pv - refl
        yu = torch.zeros_like(v)
        yu[nI - 1] = -sv[nI - 1]
        for i in range(nI - 1, 0, -1):  # sweep_up, slab i = cell i, rows 0, 1
            wv = bs(i, [None, None, yu[i, 0], yu[i, 1]], (R0, R1))
            yu[i - 1, 0] = wv[0] - sv[i - 1, 0]
            yu[i - 1, 1] = wv[1] - sv[i - 1, 1]
        return torch.cat([yd.reshape(2 * nI * w, -1), yu.reshape(2 * nI * w, -1)])

    eye = torch.eye(n, dtype=torch.complex128, device=dev)
    Pm = pre(eye)
    Bm = pre(op(eye))
    return Pm, Bm


def inner_sstep_operators(Pm, Bm):
    """``(S1, S2) = (E Pm, E^2 Pm)`` with ``E = Bm - I`` (``Bm = pre o op``): applied to the inner rhs they
    give ``E b`` and ``E^2 b`` for ``b = pre(rhs)`` in the same pass as ``b`` itself.  The shifted powers span
    the Krylov spaces of the first two GMRES steps (``span{b, A b, A^2 b}``, ``A = E + I``) and, with
    ``A V = E V + V``, let the device run those two Arnoldi steps without waiting for a product in between;
    ``E`` is small where the preconditioner works, so no large vectors cancel."""
    n = Pm.shape[0]
    E = Bm - torch.eye(n, dtype=Bm.dtype, device=Bm.device)
    S1 = E @ Pm
    S2 = E @ S1
    return S1, S2


def inner_lu_inverse(lf):
    """Direct inner backend (``_InnerLU``, ``nested.py:156-254``): the assembled cell-interface system
    ``A x = b`` with 2w x 2w blocks per interface i (unknowns: rows n of cell i and 1 of cell i+1)

    * diag  ``[[I - G_i(n,vn), -G_i(n,vnp)], [-G_i+1(1,v0), I - G_i+1(1,v1)]]``
    * lower ``[[-G_i(n,v0), -G_i(n,v1)], [0, 0]]`` at block (i, i-1)
    * upper ``[[0, 0], [-G_i+1(1,vn), -G_i+1(1,vnp)]]`` at block (i, i+1)

    is inverted once (the reference factors it by unpivoted block LU and substitutes per solve; the
    inverse applies the same linear map in one dense product, rounding order aside)."""
    cells = lf.cells
    nI = len(cells) - 1
    if nI <= 0:
        return None
    w = lf.w
    dev = cells[0].green.device
    G = [cf.green.transpose(-1, -2) for cf in cells]  # row-major G[c][row][slot]
    R1, RN = 1, 2
    V0, V1, VN, VNP = 0, 1, 2, 3
    m = 2 * nI * w
    A = torch.zeros((m, m), dtype=torch.complex128, device=dev)
    eye = torch.eye(w, dtype=torch.complex128, device=dev)
    for i in range(nI):
        gi, gp = G[i], G[i + 1]
        a, b = 2 * i * w, 2 * i * w + w
        A[a:b, a:b] = eye - gi[RN, VN]
        A[a:b, b:b + w] = -gi[RN, VNP]
        A[b:b + w, a:b] = -gp[R1, V0]
        A[b:b + w, b:b + w] = eye - gp[R1, V1]
        if i >= 1:
            A[a:b, a - 2 * w:a - w] = -gi[RN, V0]
            A[a:b, a - w:a] = -gi[RN, V1]
        if i <= nI - 2:
            A[b:b + w, b + w:b + 2 * w] = -gp[R1, VN]
            A[b:b + w, b + 2 * w:b + 3 * w] = -gp[R1, VNP]
    return torch.linalg.inv(A).contiguous()


def _scalar_blocks(H, nb, w, what):
    """Split a block-tridiagonal operator with ``nb`` blocks of width ``w`` into the shared in-block tridiagonal
    ``tw = (lower, 0, upper)``, the diagonal ``(nb, w)`` and the scalar block couplings ``lz``/``uz`` (blocks
    ``l_k I`` / ``u_k I``): the structure of the reference's FD operators (``discretization.py:223-251``).
    Raises ``ValueError`` when ``H`` is not of that form (e.g. the Q1 discretization)."""
    import scipy.sparse as sp

    H = sp.csr_matrix(H)
    if H.shape != (nb * w, nb * w):
        raise ValueError(f"{what}: operator of shape {H.shape}, expected {(nb * w, nb * w)}")
    diag = np.asarray(H.diagonal(), dtype=np.complex128).reshape(nb, w)
    i = np.arange(1, w)
    lower = np.zeros(w, dtype=np.complex128)
    upper = np.zeros(w, dtype=np.complex128)
    lower[1:] = np.asarray(H[i, i - 1]).ravel()
    upper[:-1] = np.asarray(H[i - 1, i]).ravel()
    k = np.arange(1, nb)
    lz = np.zeros(nb, dtype=np.complex128)
    uz = np.zeros(nb, dtype=np.complex128)
    lz[1:] = np.asarray(H[k * w, (k - 1) * w]).ravel()
    uz[:-1] = np.asarray(H[(k - 1) * w, k * w]).ravel()
    rebuilt = (sp.kron(sp.eye(nb), sp.diags([lower[1:], upper[:-1]], [-1, 1], shape=(w, w)))
               + sp.diags(diag.ravel()) + sp.kron(sp.diags([lz[1:], uz[:-1]], [-1, 1], shape=(nb, nb)), sp.eye(w)))
    err = abs(H - rebuilt).max()
    if err > 1e-12 * abs(H).max():
        raise ValueError(f"{what}: not a block-tridiagonal operator with scalar couplings (mismatch {err:.3e})")
    return (lower, np.zeros(w, dtype=np.complex128), upper), diag, lz, uz


def _reference_cells(ref, nxc_list, w, npml):
    """Per-cell operators (cell frame: block rows = original x, width = layer depth) of one reference layer:
    ``NestedLayerSolver.cells[c].H`` (``nested.py:297-302``) or, for a direct ``LayerWorkspace`` layer
    (Lc = 1), its own operator with the x <-> z swap applied to the unknown ordering (``nested.py:45-47``)."""
    if hasattr(ref, "cells"):
        return [cell.H for cell in ref.cells]
    wx = ref.grid.wx
    wz = ref.grid.wz
    perm = (np.arange(w)[None, :] * wx + np.arange(wx)[:, None]).ravel()  # cell (k=x, i=z) <- layer z*wx + x
    assert wz == w and len(nxc_list) == 1
    Hc = ref.H.tocsr()[perm][:, perm]
    return [Hc]


def _k1_layer_operators(grid, lf, Lc, cext, coffs, device, green, q0, ref):
    """Green blocks, sampled trace responses and pass-0 operators of one layer's cells as many-RHS solves with
    the repo's own cell-solve kernel K1 (``csrc/k1_cell_solve.cu`` through ``pt_cell_solve_device``).

    This is ``GreenBlockSet.build`` (``green.py:103-129``, called per cell at ``nested.py:303-307``): the
    reference solves ``H_c x = coef_slot e_j`` at the slot row for the ``w`` unit vectors of each of the four
    slots with the cell's SuperLU factors (``subdomain.py:205-221``); here the ``4 w`` unit sources of a cell are
    one K1 launch on the twisted Schur factors already resident on the device (a one-layer, factor-only context:
    ``pt_problem.green == NULL``), and the blocks are row samples of the solutions.  The operators of the online
    restructuring come from the same solves (``gsmp``: every block row of those solutions at the layer trace
    rows) and from a second launch (``q0``: the ``4 nk`` layer slot sources of the kept block rows).
    """
    import ctypes as C

    from . import _abi

    npml, w, n = grid.npml, lf.w, lf.n
    wx = grid.nx + 2 * npml
    zx = np.zeros(wx, dtype=np.complex128)
    zz = np.zeros(w, dtype=np.complex128)
    one = Factors(grid.nx, n, grid.h, npml, 0.0, 1, Lc, [lf], cext, coffs, (zx, zx, zx), (zz, zz, zz),
                  np.zeros((w, wx)))
    ctx = _abi.Context(one, device=device.index if device.index is not None else torch.cuda.current_device())
    L_ = _abi.lib()
    try:
        jrows = [npml - 1, npml, n + npml - 1, n + npml]  # layer trace rows 0, 1, n, n+1 inside a block row
        for ci, cf in enumerate(lf.cells):
            wzc, nxc = cf.wzc, cf.nxc
            rows4 = [int(r) for r in (cf.krows[1], cf.krows[0], cf.krows[3], cf.krows[2])]  # r0, r1, rn, rnp
            ar = torch.arange(w, device=device)

            def solve(B):
                X = torch.empty_like(B)
                rc = L_.pt_cell_solve_device(ctx.handle, 0, ci, C.c_void_p(B.data_ptr()), B.shape[0],
                                             C.c_void_p(X.data_ptr()))
                if rc != _abi.PT_OK:
                    raise RuntimeError(f"pt_cell_solve_device failed ({rc}): {_abi.last_error()}")
                return X

            if green:
                # right-hand side (slot s, column a): coef_s e_a at block row krow_s; K1 volumes are [rhs][wz_c][w]
                B = torch.zeros((4, w, wzc, w), dtype=torch.complex128, device=device)
                for s in range(4):
                    B[s, ar, int(cf.krows[s]), ar] = complex(cf.coefs[s])
                torch.cuda.synchronize(device)
                X = solve(B.view(4 * w, wzc, w)).view(4, w, wzc, w)
                del B
                if ref is not None and hasattr(ref, "blocksets"):
                    bs = ref.blocksets[ci]  # the reference's own GreenBlockSet matrices (green.py:103-129)
                    cf.green = torch.stack([torch.stack([torch.as_tensor(
                        np.asarray(bs.dense(jrow, slot)).T, dtype=torch.complex128, device=device)
                        for slot in SLOTS]) for jrow in (0, 1, nxc, nxc + 1)]).contiguous()
                else:
                    # column-major block (row j, slot s): element (i, a) at a * w + i = X[s, a, row_j, i]
                    cf.green = X[:, :, rows4, :].permute(2, 0, 1, 3).contiguous()
                cf.gsmp = X[:, :, :, jrows].permute(2, 3, 0, 1).contiguous()  # (wzc, 4 trace rows, 4 slots, w)
                del X
            if q0:
                lo = 0 if ci == 0 else npml
                hi = wzc if ci == Lc - 1 else npml + nxc
                nk = hi - lo
                nk4 = (nk + 3) // 4 * 4
                kk = torch.arange(nk, device=device)
                B = torch.zeros((4, nk, wzc, w), dtype=torch.complex128, device=device)
                for s in range(4):  # layer slot source s at kept block row lo + kk: coef_s at layer row prow_s
                    B[s, kk, lo + kk, int(lf.prows[s])] = complex(lf.coefs[s])
                torch.cuda.synchronize(device)
                X = solve(B.view(4 * nk, wzc, w)).view(4, nk, wzc, w)
                del B
                qt = X[:, :, rows4, :].permute(2, 3, 0, 1).reshape(4 * w, 4, nk)
                qs = X[:, :, lo:hi, :][:, :, :, jrows].permute(2, 3, 0, 1).reshape(4 * nk, 4, nk)
                m = 4 * w + 4 * nk
                mp = (m + 7) // 8 * 8
                q = torch.zeros((mp, 4, nk4), dtype=torch.complex128, device=device)
                q[:m, :, :nk] = torch.cat([qt, qs])
                cf.q0 = q.reshape(mp, 4 * nk4)
                del X
    finally:
        ctx.close()


def _batched_twisted_factors(grid, model, pml, partition, Lc, cext, coffs, device, tm, budget=24e9):
    """Twisted Schur factors of every cell, the recursion batched over ALL cells of equal shape (layer depth n,
    cell extent nx_c) across the layers: the block couplings depend only on (n, nx_c), so a config has a handful
    of shapes (cfg5: 4) and the ``wz_c`` dependent inversion steps run on hundreds of cells at once instead of
    once per layer.  Returns ``{(layer, cell): (wz_c, w, w) column-major twisted factors}``; ``budget`` bounds the
    bytes of one batch's temporaries."""
    npml, h, omega = grid.npml, grid.h, pml.omega
    c = np.asarray(model.c, dtype=float)
    shapes = {}
    for ell, (n, off) in enumerate(zip(partition.extents, partition.offsets)):
        for ci, nxc in enumerate(cext):
            shapes.setdefault((n, nxc), []).append((ell, off, ci))
    out = {}
    for (n, nxc), lst in shapes.items():
        w, wzc = n + 2 * npml, nxc + 2 * npml
        if wzc < 3:
            raise ValueError("cells need at least 3 block rows (nx_c + 2 npml >= 3)")
        tw = axis_tridiag(pml, n, h)
        lz, tzm, uz = axis_tridiag(pml, nxc, h)
        per = 3.0 * wzc * w * w * 16
        maxb = max(1, int(budget // per))
        for b0 in range(0, len(lst), maxb):
            part = lst[b0 : b0 + maxb]
            diag = np.empty((len(part), wzc, w), dtype=np.complex128)
            for b, (ell, off, ci) in enumerate(part):
                cc = c[off : off + w, coffs[ci] : coffs[ci] + wzc].T  # (wzc, w): the transposed layer's cell
                diag[b] = tzm[:, None] - omega**2 * (1.0 / cc**2)
            dg = torch.as_tensor(diag, device=device)
            tm.mark()
            sinv = _schur_inverses(tw, dg, lz, uz, device)
            tm.mark("schur")
            tinv = _twisted_inverses(tw, dg, lz, uz, sinv, device)
            del sinv
            cm = tinv.transpose(-1, -2).contiguous()
            del tinv
            tm.mark("twisted")
            for b, (ell, off, ci) in enumerate(part):
                out[(ell, ci)] = cm[b]
    return out


def build_factors(grid, model, pml, partition, Lc, device="cpu", green=True, q0=None, inner_dense=None,
                  backend="pt", reference_layers=None, cell_solver=None):
    """Offline stage for a partitioned problem (all layers, all cells).

    ``grid``/``model``/``pml``/``partition`` follow the reference value types
    (``discretization.py:58-220``, ``subdomain.py:51-73``).

    ``cell_solver``: ``"k1"`` runs the unit-source cell solves of the Green blocks and of the pass-0 /
    sampled-response operators on the device with the online stage's own K1 kernel (default on a CUDA device);
    ``"torch"`` runs them as torch block substitutions (default on the CPU; the parity check of the K1 route).

    ``reference_layers``: the reference's own ``build_nested_layers`` output (``NestedLayerSolver`` objects,
    ``nested.py:272-319``) or its direct ``LayerWorkspace`` layers (``subdomain.py:202-236``, Lc = 1).  The
    couplings are then read from the layers' assembled operators (``LayerOperator.H``, the cells' ``H``) and
    the interface Green blocks are the reference's own ``GreenBlockSet`` matrices (``green.py:90-153``),
    uploaded as they are; only the device-side factorisation (Schur inverses) and the operators of the
    online restructuring are computed here.
    """
    device = torch.device(device)
    if cell_solver is None:
        cell_solver = "k1" if device.type == "cuda" else "torch"
    if cell_solver not in ("k1", "torch"):
        raise ValueError(f"unknown cell_solver {cell_solver!r}")
    if cell_solver == "k1" and device.type != "cuda":
        raise ValueError("cell_solver='k1' needs a CUDA device (the B200 kernels have no CPU fallback)")
    use_k1 = cell_solver == "k1"
    if q0 is None:
        q0 = green
    if inner_dense is None:
        # dense pre / pre.op matrices cost 128 (Lc-1)^2 w^2 flops per inner product against the Green-block
        # programs' O(Lc w^2): one product wins up to Lc = 8 (measured on cfg2 and cfg3); the memory
        # (2 (4 (Lc-1) w)^2 per layer) also grows with (Lc-1)^2
        inner_dense = green and Lc <= 8
    npml, h, omega = grid.npml, grid.h, pml.omega
    tm = _Timer(device)
    cext = _split(grid.nx, Lc)  # partition_layers(sgrid, Lc), nested.py:294-296
    coffs = tuple(int(v) for v in np.concatenate([[0], np.cumsum(cext)[:-1]]))
    c = np.asarray(model.c, dtype=float)
    # device route: every cell's factors first, batched by cell shape across the layers
    pre = None
    if use_k1 and reference_layers is None:
        pre = _batched_twisted_factors(grid, model, pml, partition, Lc, cext, coffs, device, tm)
    layers = []
    for ell, (n, off) in enumerate(zip(partition.extents, partition.offsets)):
        w = n + 2 * npml
        # layer-level cut couplings: the layer's own depth axis (subdomain.py:157-182)
        ref = reference_layers[ell] if reference_layers is not None else None
        if ref is None:
            lzL, _, uzL = axis_tridiag(pml, n, h)
        else:  # the layer's depth-axis couplings H[(z, x), (z -/+ 1, x)] at x = 0 (discretization.py:251)
            HL = ref.H.tocsr()
            wxl = ref.grid.wx
            z = np.arange(1, w)
            lzL = np.zeros(w, dtype=np.complex128)
            uzL = np.zeros(w, dtype=np.complex128)
            lzL[1:] = np.asarray(HL[z * wxl, (z - 1) * wxl]).ravel()
            uzL[:-1] = np.asarray(HL[(z - 1) * wxl, z * wxl]).ravel()
            ref_ops = _reference_cells(ref, cext, w, npml)
        lcoefs, lrows = cut_coefs(lzL, uzL, npml, n)
        lf = LayerFactors(ell, n, off, w, lcoefs, lrows)
        c_layer = c[off : off + w, :]  # VelocityModel.restrict (subdomain.py:233-234)
        # group cells of equal nx_c for batched factorization
        groups = {}
        for ci, nxc in enumerate(cext):
            groups.setdefault(nxc, []).append(ci)
        cells = [None] * Lc
        for nxc, idxs in groups.items():
            wzc = nxc + 2 * npml
            if pre is not None:
                lz, _, uz = axis_tridiag(pml, nxc, h)
                ccoefs, ckrows = cut_coefs(lz, uz, npml, nxc)
                for ci in idxs:
                    cells[ci] = CellFactors(ell, ci, w, wzc, nxc, coffs[ci], pre.pop((ell, ci)), np.asarray(lz),
                                            np.asarray(uz), None, ccoefs, ckrows, None, None)
                continue
            diag = np.empty((len(idxs), wzc, w), dtype=np.complex128)
            if ref is None:
                lz, tzm, uz = axis_tridiag(pml, nxc, h)  # along block rows (original x)
                for b, ci in enumerate(idxs):
                    # cell model: transposed layer restricted to rows [off_c, off_c+wzc)
                    cc = c_layer[:, coffs[ci] : coffs[ci] + wzc].T  # (wzc, w)
                    diag[b] = tzm[:, None] - omega**2 * (1.0 / cc**2)
            else:
                parts = [_scalar_blocks(ref_ops[ci], wzc, w, f"layer {ell + 1} cell {ci + 1}") for ci in idxs]
                tw, _, lz, uz = parts[0]
                for b, (twb, db, lzb, uzb) in enumerate(parts):
                    if not (np.allclose(twb[0], tw[0], rtol=0, atol=0) and np.array_equal(lzb, lz)
                            and np.array_equal(uzb, uz)):
                        raise ValueError("cells of equal width must share their couplings")
                    diag[b] = db
            ccoefs, ckrows = cut_coefs(lz, uz, npml, nxc)
            dg = torch.as_tensor(diag, device=device)
            if ref is None:
                tw = axis_tridiag(pml, n, h)  # across the cell block: the layer depth
            tm.mark()
            sinv = _schur_inverses(tw, dg, lz, uz, device)
            tm.mark("schur")
            gblk = None
            gsmp = None
            if green and not use_k1:
                # H_c^{-1} columns at the four slot rows, sampled at the four rows
                rows4 = [int(r) for r in (ckrows[1], ckrows[0], ckrows[3], ckrows[2])]  # r0,r1,rn,rnp
                eye = torch.eye(w, dtype=torch.complex128, device=device)
                rhs = torch.zeros((len(idxs), wzc, w, 4 * w), dtype=torch.complex128,
                                  device=device)
                for s in range(4):
                    rhs[:, int(ckrows[s]), :, s * w : (s + 1) * w] = complex(ccoefs[s]) * eye
                X = _block_solve(sinv, lz, uz, rhs)
                gblk = torch.empty((len(idxs), 4, 4, w, w), dtype=torch.complex128,
                                   device=device)
                if ref is not None and hasattr(ref, "blocksets"):
                    # the reference's own GreenBlockSet matrices (green.py:103-129), rows j = 0, 1, n, n+1
                    for b, ci in enumerate(idxs):
                        bs = ref.blocksets[ci]
                        for jr, jrow in enumerate((0, 1, nxc, nxc + 1)):
                            for s, slot in enumerate(SLOTS):
                                gblk[b, jr, s] = torch.as_tensor(
                                    np.asarray(bs.dense(jrow, slot)).T, dtype=torch.complex128, device=device)
                else:
                    for jr, rr in enumerate(rows4):
                        for s in range(4):
                            # column-major storage == transpose of the row-major block
                            gblk[:, jr, s] = X[:, rr, :, s * w : (s + 1) * w].transpose(-1, -2)
                # layer trace rows 0, 1, n, n+1 in the cell-local frame (offset npml - 1), every block row
                jrows = [npml - 1, npml, n + npml - 1, n + npml]
                gsmp = X[:, :, jrows, :].reshape(len(idxs), wzc, 4, 4, w).contiguous()
                del X, rhs
            q0c = [None] * len(idxs)
            if q0 and not use_k1:
                # responses to the layer slot sources at every block row: K_full = 4 wzc columns
                rows4 = [int(r) for r in (ckrows[1], ckrows[0], ckrows[3], ckrows[2])]  # r0,r1,rn,rnp
                jrows = [npml - 1, npml, n + npml - 1, n + npml]
                kf = torch.arange(wzc, device=device)
                rhs = torch.zeros((len(idxs), wzc, w, 4 * wzc), dtype=torch.complex128, device=device)
                for s in range(4):
                    rhs[:, kf, int(lrows[s]), s * wzc + kf] = complex(lcoefs[s])
                X = _block_solve(sinv, lz, uz, rhs)
                del rhs
                for b, ci in enumerate(idxs):
                    lo = 0 if ci == 0 else npml
                    hi = wzc if ci == Lc - 1 else npml + nxc
                    nk = hi - lo
                    nk4 = (nk + 3) // 4 * 4  # slot column blocks padded to whole DMMA k-steps
                    cols = torch.cat([s * wzc + torch.arange(lo, hi, device=device) for s in range(4)])
                    qt = X[b][rows4][:, :, cols].reshape(4 * w, 4, nk)
                    qs = X[b][lo:hi][:, jrows][:, :, cols].reshape(4 * nk, 4, nk)
                    m = 4 * w + 4 * nk
                    mp = (m + 7) // 8 * 8
                    q = torch.zeros((mp, 4, nk4), dtype=torch.complex128, device=device)
                    q[:m, :, :nk] = torch.cat([qt, qs])
                    q0c[b] = q.reshape(mp, 4 * nk4)
                del X
            if wzc < 3:
                raise ValueError("cells need at least 3 block rows (nx_c + 2 npml >= 3)")
            tm.mark("torch-operators")
            tinv = _twisted_inverses(tw, dg, lz, uz, sinv, device)
            tm.mark("twisted")
            sinv_cm = tinv.transpose(-1, -2).contiguous()
            for b, ci in enumerate(idxs):
                cells[ci] = CellFactors(
                    ell, ci, w, wzc, nxc, coffs[ci], sinv_cm[b],
                    np.asarray(lz), np.asarray(uz),
                    None if gblk is None else gblk[b].contiguous(),
                    ccoefs, ckrows,
                    None if gsmp is None else gsmp[b].contiguous(),
                    q0c[b],
                )
        lf.cells = cells
        if use_k1 and (green or q0):
            if pre is None:
                del sinv, tinv, sinv_cm, dg
            tm.mark()
            _k1_layer_operators(grid, lf, Lc, cext, coffs, device, green, q0, ref)
            tm.mark("k1-operators")
        if green and backend == "lu":
            lf.lu_inv = inner_lu_inverse(lf)
        elif green and inner_dense:
            ops = inner_dense_operators(lf)
            if ops is not None:
                # [pre, pre o op, E pre, E^2 pre]: the last two drive the s-step start of the inner GMRES
                lf.dense = torch.stack(list(ops) + list(inner_sstep_operators(*ops))).contiguous()
        layers.append(lf)
    tm.report()
    tx = axis_tridiag(pml, grid.nx, h)
    tz = axis_tridiag(pml, grid.nz, h)
    return Factors(grid.nx, grid.nz, h, npml, omega, partition.L, Lc, layers, cext, coffs,
                   tx, tz, 1.0 / c**2)


def residual_from_operator(H, wz, wx):
    """``(tx, tz, hdiag)`` of an assembled global 5-point operator (``PolarizedTracesSolver(global_operator=H)``,
    ``sie.py:381, 387-390``) for the device residual ``||H u - f|| / ||f||`` (``sie.py:441-445``): the x / z
    neighbour couplings (row-independent / column-independent in the FD operator, ``discretization.py:251``) and
    the full complex diagonal.  Raises ``ValueError`` if ``H`` is not of that form."""
    import scipy.sparse as sp

    H = sp.csr_matrix(H)
    n = wz * wx
    if H.shape != (n, n):
        raise ValueError(f"global_operator has shape {H.shape}, the grid needs {(n, n)}")
    x = np.arange(1, wx)
    txl = np.zeros(wx, dtype=np.complex128)
    txu = np.zeros(wx, dtype=np.complex128)
    txl[1:] = np.asarray(H[x, x - 1]).ravel()
    txu[:-1] = np.asarray(H[x - 1, x]).ravel()
    z = np.arange(1, wz)
    tzl = np.zeros(wz, dtype=np.complex128)
    tzu = np.zeros(wz, dtype=np.complex128)
    tzl[1:] = np.asarray(H[z * wx, (z - 1) * wx]).ravel()
    tzu[:-1] = np.asarray(H[(z - 1) * wx, z * wx]).ravel()
    hdiag = np.asarray(H.diagonal(), dtype=np.complex128).reshape(wz, wx)
    rebuilt = (sp.kron(sp.eye(wz), sp.diags([txl[1:], txu[:-1]], [-1, 1], shape=(wx, wx)))
               + sp.kron(sp.diags([tzl[1:], tzu[:-1]], [-1, 1], shape=(wz, wz)), sp.eye(wx))
               + sp.diags(hdiag.ravel()))
    err = abs(H - rebuilt).max()
    if err > 1e-12 * abs(H).max():
        raise ValueError(f"global_operator is not a 5-point FD operator (mismatch {err:.3e})")
    zeros_x = np.zeros(wx, dtype=np.complex128)
    zeros_z = np.zeros(wz, dtype=np.complex128)
    return (txl, zeros_x, txu), (tzl, zeros_z, tzu), hdiag
