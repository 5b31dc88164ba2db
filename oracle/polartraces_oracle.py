"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain numpy/scipy restatement of the reference's online nested
polarized-traces path (``backend="pt"``, ``assembled_boundary=False``), used
only as the checker by ``tests/``, ``__graft_entry__.smoke()`` and the CPU legs
of ``bench.py``.  The product (``paper_1510_01831_b200``) never imports it.

Every function cites the reference lines it follows
(``/root/reference/pkg/src/polartraces/...``).  Third-party arithmetic is the
same as the reference's: SuperLU via ``scipy.sparse.linalg.splu`` (scipy is
unpinned upstream, ``pkg/pyproject.toml:12``; 1.18.1 in this image) and BLAS
via numpy.

Pinning: ``tests/golden/make_golden.py`` runs the live reference (importable in
the build container only) on small problems and on config 1 and commits the
results as fixtures; ``tests/test_oracle_golden.py`` checks this module against
them, and against the SURVEY.md section 8(c) known-answer anchors.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "fd_operator",
    "Local",
    "gmres",
    "NestedLayer",
    "OracleSolver",
    "OracleResult",
    "KrylovBreakdown",
    "InnerSolveError",
]


class KrylovBreakdown(RuntimeError):
    """``krylov.py:42-46``."""

    def __init__(self, message, basis_size=None, residuals=None):
        super().__init__(message)
        self.basis_size = basis_size
        self.residuals = residuals or []


class InnerSolveError(RuntimeError):
    """``nested.py:50-51``."""


# --------------------------------------------------------------------------
# discretization (discretization.py:149-176, 223-251)


def _alpha_axis(n, npml, h, C, omega, half):
    coords = h * (np.arange(1 - npml, n + npml + 1, dtype=float) + half)
    span = (n + 1) * h
    sig = np.zeros_like(coords)
    if npml > 0:
        d = npml * h
        lo = coords < 0.0
        hi = coords > span
        sig[lo] = (C / d) * (coords[lo] / d) ** 2
        sig[hi] = (C / d) * ((coords[hi] - span) / d) ** 2
    return 1.0 / (1.0 + 1j * sig / omega)


def fd_operator(nx, nz, h, npml, c, C, omega):
    """5-point PML Helmholtz operator on the extended grid, CSR.

    ``discretization.py:223-251``: ``kron(I_z, T_x) + kron(T_z, I_x) - omega^2 diag(m)``.
    """
    h2 = h * h

    def tri(n):
        a0 = _alpha_axis(n, npml, h, C, omega, 0.0)
        ap = _alpha_axis(n, npml, h, C, omega, +0.5)
        am = _alpha_axis(n, npml, h, C, omega, -0.5)
        return sp.diags(
            [-(a0 * am / h2)[1:], a0 * (ap + am) / h2, -(a0 * ap / h2)[:-1]],
            offsets=[-1, 0, 1], format="csr",
        )

    wx, wz = nx + 2 * npml, nz + 2 * npml
    m = 1.0 / np.asarray(c, dtype=float) ** 2
    return (
        sp.kron(sp.identity(wz, format="csr"), tri(nx))
        + sp.kron(tri(nz), sp.identity(wx, format="csr"))
        - sp.diags(omega**2 * m.ravel())
    ).tocsr()


def split_extents(n, parts):
    """``subdomain.py:88-90``: near-equal parts, remainder first."""
    base, rem = divmod(n, parts)
    return tuple(base + 1 if i < rem else base for i in range(parts))


def _offsets(extents):
    return tuple(int(v) for v in np.concatenate([[0], np.cumsum(extents)[:-1]]))


# --------------------------------------------------------------------------
# a factorized local problem (subdomain.py:113-224)


class Local:
    """One slab (layer or cell) with its own absorbing collar.

    ``nx`` points across, ``n`` interior depth rows, extended ``(wz, wx)``.
    """

    def __init__(self, nx, n, h, npml, c, C, omega):
        self.nx, self.n, self.h, self.npml = nx, n, h, npml
        self.wx, self.wz = nx + 2 * npml, n + 2 * npml
        self.width = self.wx
        self.shape = (self.wz, self.wx)
        self.H = fd_operator(nx, n, h, npml, c, C, omega)
        self.lu = spla.splu(self.H.tocsc())  # subdomain.py:208
        self._blk = {}

    def row(self, k):  # subdomain.py:133-138
        r = k + self.npml - 1
        if not 0 <= r < self.wz:
            raise ValueError(f"depth {k} outside local extended grid")
        return r

    def block(self, j, k):  # subdomain.py:147-154
        if (j, k) not in self._blk:
            rj = np.arange(self.row(j) * self.wx, (self.row(j) + 1) * self.wx)
            rk = np.arange(self.row(k) * self.wx, (self.row(k) + 1) * self.wx)
            self._blk[(j, k)] = self.H[rj][:, rk].tocsr()
        return self._blk[(j, k)]

    def solve(self, rhs):  # subdomain.py:214-221
        a = np.asarray(rhs, dtype=complex)
        if a.shape == self.shape:
            return self.lu.solve(a.ravel()).reshape(self.shape)
        return self.lu.solve(a)

    def add_sources(self, rhs, v0, v1, vn, vnp):
        """src_top then src_bot (``subdomain.py:157-182``), in place."""
        n = self.n
        if v0 is not None:
            rhs[self.row(1)] -= self.block(1, 0) @ v0
        if v1 is not None:
            rhs[self.row(0)] += self.block(0, 1) @ v1
        if vn is not None:
            rhs[self.row(n + 1)] += self.block(n + 1, n) @ vn
        if vnp is not None:
            rhs[self.row(n)] -= self.block(n, n + 1) @ vnp
        return rhs

    def boundary_samples(self, v0, v1, vn, vnp, rows):  # subdomain.py:184-194
        rhs = self.add_sources(np.zeros(self.shape, dtype=complex), v0, v1, vn, vnp)
        w = self.solve(rhs)
        return [w[self.row(r)].copy() for r in rows]

    def newton_samples(self, f, rows):  # subdomain.py:196-199
        w = self.solve(f)
        return [w[self.row(r)].copy() for r in rows]


# --------------------------------------------------------------------------
# GMRES (krylov.py:53-135)


def gmres(op, rhs, precond, ktol, max_iter, restart=0):
    """Left-preconditioned GMRES, MGS Arnoldi, complex Givens, x0 = 0.

    Returns ``(x, iterations, residuals, converged)``.
    """
    b = precond(np.asarray(rhs, dtype=complex))
    n = b.size
    beta0 = np.linalg.norm(b)
    if beta0 == 0.0:
        return np.zeros(n, dtype=complex), 0.0, [0.0], True
    x = np.zeros(n, dtype=complex)
    cycle = restart if restart > 0 else max_iter
    hist = []
    total = 0
    while total < max_iter:
        r = b - precond(op(x)) if total > 0 else b.copy()
        beta = np.linalg.norm(r)
        if beta / beta0 <= ktol:
            hist.append(beta / beta0)
            return x, float(total), hist, True
        m = min(cycle, max_iter - total)
        V = np.zeros((m + 1, n), dtype=complex)
        V[0] = r / beta
        Hs = np.zeros((m + 1, m), dtype=complex)
        cs = np.zeros(m, dtype=complex)
        sn = np.zeros(m, dtype=complex)
        g = np.zeros(m + 1, dtype=complex)
        g[0] = beta
        k = 0
        for j in range(m):
            w = precond(op(V[j]))
            for i in range(j + 1):
                Hs[i, j] = np.vdot(V[i], w)
                w -= Hs[i, j] * V[i]
            hn = np.linalg.norm(w)
            Hs[j + 1, j] = hn
            for i in range(j):
                t = cs[i] * Hs[i, j] + sn[i] * Hs[i + 1, j]
                Hs[i + 1, j] = -np.conj(sn[i]) * Hs[i, j] + np.conj(cs[i]) * Hs[i + 1, j]
                Hs[i, j] = t
            d = np.sqrt(abs(Hs[j, j]) ** 2 + hn**2)
            if d == 0.0:
                raise KrylovBreakdown("zero Hessenberg column", j + 1, hist)
            cs[j] = np.conj(Hs[j, j]) / d
            sn[j] = hn / d
            Hs[j, j] = cs[j] * Hs[j, j] + sn[j] * hn
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            k = j + 1
            res = abs(g[j + 1]) / beta0
            hist.append(res)
            if hn == 0.0:
                if res > ktol:
                    raise KrylovBreakdown("happy breakdown before convergence", k, hist)
                break
            V[j + 1] = w / hn
            if res <= ktol:
                break
        y = np.zeros(k, dtype=complex)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - Hs[i, i + 1 : k] @ y[i + 1 : k]) / Hs[i, i]
        x = x + V[:k].T @ y
        if hist[-1] <= ktol:
            return x, float(total), hist, True
    return x, float(total), hist, False


def bicgstab(op, rhs, precond, ktol, max_iter):
    """Left-preconditioned BiCGstab, half steps counted as 0.5 iterations, shadow residual = the
    initial preconditioned residual, x0 = 0 (krylov.py:138-201).

    Returns ``(x, iterations, residuals, converged)``; breakdowns raise ``KrylovBreakdown``.
    """
    b = precond(np.asarray(rhs, dtype=complex))
    n = b.size
    beta0 = np.linalg.norm(b)
    if beta0 == 0.0:
        return np.zeros(n, dtype=complex), 0.0, [0.0], True

    def pa(v):
        return precond(op(v))

    x = np.zeros(n, dtype=complex)
    r = b.copy()
    r0 = r.copy()
    rho = alpha = omega = 1.0 + 0.0j
    v = np.zeros(n, dtype=complex)
    p = np.zeros(n, dtype=complex)
    hist = [np.linalg.norm(r) / beta0]
    count = 0.0
    for _ in range(int(np.ceil(max_iter))):
        rho_new = np.vdot(r0, r)
        if abs(rho_new) < 1e-300 * beta0**2:
            raise KrylovBreakdown("BiCGstab breakdown (rho ~ 0)", count, hist)
        beta = (rho_new / rho) * (alpha / omega) if count > 0 else 0.0
        rho = rho_new
        p = r + beta * (p - omega * v) if count > 0 else r.copy()
        v = pa(p)
        denom = np.vdot(r0, v)
        if abs(denom) < 1e-300 * beta0**2:
            raise KrylovBreakdown("BiCGstab breakdown (r0.v ~ 0)", count, hist)
        alpha = rho / denom
        s = r - alpha * v
        count += 0.5
        res = np.linalg.norm(s) / beta0
        hist.append(res)
        if res <= ktol:
            return x + alpha * p, count, hist, True
        t = pa(s)
        tt = np.vdot(t, t)
        if abs(tt) == 0.0:
            raise KrylovBreakdown("BiCGstab breakdown (t = 0)", count, hist)
        omega = np.vdot(t, s) / tt
        x = x + alpha * p + omega * s
        r = s - omega * t
        count += 0.5
        res = np.linalg.norm(r) / beta0
        hist.append(res)
        if res <= ktol:
            return x, count, hist, True
        if count >= max_iter:
            break
    return x, count, hist, False


# --------------------------------------------------------------------------
# trace machinery over a list of slabs (sie.py:112-346)


class Traces:
    """Interface operators of one decomposition level.

    ``slabs`` are objects with ``n``, ``width``, ``npml``, ``wz``,
    ``boundary_samples``, ``newton_samples``, ``add_sources`` and ``solve``;
    ``offsets`` are the slabs' interior offsets along the stacking direction.
    """

    def __init__(self, slabs, offsets):
        self.slabs = list(slabs)
        self.offsets = offsets
        self.L = len(self.slabs)
        self.nI = self.L - 1
        self.w = self.slabs[0].width

    def keep_range(self, ell):  # sie.py:146-147, 343-344
        s = self.slabs[ell - 1]
        lo = 0 if ell == 1 else s.npml
        hi = s.wz if ell == self.L else s.npml + s.n
        return lo, hi

    def split(self, f):  # sie.py:134-151
        out = []
        for ell, s in enumerate(self.slabs, start=1):
            off = self.offsets[ell - 1]
            loc = np.array(f[off : off + s.wz], dtype=complex)
            lo, hi = self.keep_range(ell)
            loc[:lo] = 0.0
            loc[hi:] = 0.0
            out.append(loc)
        return out

    def newton_rhs(self, f_locals):
        """``newton_tables`` + ``build_rhs_polarized`` (sie.py:175-188, 230-242)."""
        down = np.zeros((self.nI, 2, self.w), dtype=complex)
        up = np.zeros((self.nI, 2, self.w), dtype=complex)
        for ell, s in enumerate(self.slabs, start=1):
            rows = ([0, 1] if ell >= 2 else []) + ([s.n, s.n + 1] if ell <= self.L - 1 else [])
            if not rows:
                continue
            smp = dict(zip(rows, s.newton_samples(f_locals[ell - 1], rows)))
            if ell <= self.L - 1:
                down[ell - 1, 0] = -smp[s.n]
                down[ell - 1, 1] = -smp[s.n + 1]
            if ell >= 2:
                up[ell - 2, 0] = -smp[0]
                up[ell - 2, 1] = -smp[1]
        return down, up

    def apply_M(self, d, p):  # sie.py:203-228
        od = np.zeros_like(d)
        ou = np.zeros_like(p)
        for ell, s in enumerate(self.slabs, start=1):
            top, bot = ell >= 2, ell <= self.L - 1
            it, ib = ell - 2, ell - 1
            if bot:
                v0 = d[ib - 1, 0] + p[ib - 1, 0] if top else None
                v1 = d[ib - 1, 1] + p[ib - 1, 1] if top else None
                wb = s.boundary_samples(v0, v1, p[ib, 0], p[ib, 1], (s.n, s.n + 1))
                od[ib, 0] = wb[0] - (d[ib, 0] + p[ib, 0])
                od[ib, 1] = wb[1] - d[ib, 1]
            if top:
                vn = p[ib, 0] + d[ib, 0] if bot else None
                vnp = p[ib, 1] + d[ib, 1] if bot else None
                wt = s.boundary_samples(d[it, 0], d[it, 1], vn, vnp, (0, 1))
                ou[it, 0] = wt[0] - p[it, 0]
                ou[it, 1] = wt[1] - (d[it, 1] + p[it, 1])
        return od, ou

    def sweep_down(self, v):  # sie.py:272-283
        out = np.zeros_like(v)
        if self.nI == 0:
            return out
        out[0] = -v[0]
        for i in range(2, self.nI + 1):
            s = self.slabs[i - 1]
            w = s.boundary_samples(out[i - 2, 0], out[i - 2, 1], None, None, (s.n, s.n + 1))
            out[i - 1, 0] = w[0] - v[i - 1, 0]
            out[i - 1, 1] = w[1] - v[i - 1, 1]
        return out

    def sweep_up(self, v):  # sie.py:285-296
        out = np.zeros_like(v)
        if self.nI == 0:
            return out
        out[self.nI - 1] = -v[self.nI - 1]
        for i in range(self.nI - 1, 0, -1):
            s = self.slabs[i]
            w = s.boundary_samples(None, None, out[i, 0], out[i, 1], (0, 1))
            out[i - 1, 0] = w[0] - v[i - 1, 0]
            out[i - 1, 1] = w[1] - v[i - 1, 1]
        return out

    def reflections(self, yd):  # sie.py:298-308
        out = np.zeros_like(yd)
        for i in range(1, self.nI + 1):
            s = self.slabs[i]
            b0 = yd[i, 0] if i <= self.nI - 1 else None
            b1 = yd[i, 1] if i <= self.nI - 1 else None
            w = s.boundary_samples(yd[i - 1, 0], yd[i - 1, 1], b0, b1, (0, 1))
            out[i - 1, 0] = w[0]
            out[i - 1, 1] = w[1] - yd[i - 1, 1]
        return out

    def precond(self, d, p, kind="gs"):  # sie.py:322-329
        yd = self.sweep_down(d)
        if kind == "gs":
            return yd, self.sweep_up(p - self.reflections(yd))
        return yd, self.sweep_up(p)

    def flat_ops(self, kind="gs"):
        nI, w = self.nI, self.w
        half = nI * 2 * w

        def unpack(x):
            return x[:half].reshape(nI, 2, w), x[half:].reshape(nI, 2, w)

        def op(x):
            a, b = self.apply_M(*unpack(np.asarray(x, dtype=complex)))
            return np.concatenate([a.ravel(), b.ravel()])

        def pre(x):
            a, b = self.precond(*unpack(np.asarray(x, dtype=complex)), kind=kind)
            return np.concatenate([a.ravel(), b.ravel()])

        return op, pre, unpack

    def reconstruct(self, t, f_locals, shape):  # sie.py:332-346
        out = np.zeros(shape, dtype=complex)
        for ell, s in enumerate(self.slabs, start=1):
            top = t[ell - 2] if ell >= 2 else (None, None)
            bot = t[ell - 1] if ell <= self.L - 1 else (None, None)
            rhs = s.add_sources(np.zeros(s.shape, dtype=complex), top[0], top[1], bot[0], bot[1])
            rhs += f_locals[ell - 1]
            w = s.solve(rhs)
            off = self.offsets[ell - 1]
            lo, hi = self.keep_range(ell)
            out[off + lo : off + hi] = w[lo:hi]
        return out


# --------------------------------------------------------------------------
# cells with dense Green blocks (green.py:103-153, nested.py:54-122)


SLOTS = ("v0", "v1", "vn", "vnp")


class Cell(Local):
    """A cell whose boundary application uses its 16 dense Green blocks."""

    def __init__(self, *a, counter=None):
        super().__init__(*a)
        n, w = self.n, self.width
        self.counter = counter
        eye = np.eye(w, dtype=complex)
        srcs = {  # green.py:370-377
            "v0": (1, -(self.block(1, 0) @ eye)),
            "v1": (0, self.block(0, 1) @ eye),
            "vn": (n + 1, self.block(n + 1, n) @ eye),
            "vnp": (n, -(self.block(n, n + 1) @ eye)),
        }
        self.G = {}
        for slot in SLOTS:
            k, mat = srcs[slot]
            rhs = np.zeros((self.wz * self.wx, w), dtype=complex)
            rhs.reshape(self.wz, self.wx, w)[self.row(k)] = mat
            sol = self.lu.solve(rhs)
            for j in (0, 1, n, n + 1):
                self.G[(j, slot)] = np.ascontiguousarray(
                    sol[self.row(j) * self.wx : (self.row(j) + 1) * self.wx, :]
                )

    def boundary_samples(self, v0, v1, vn, vnp, rows):  # nested.py:113-122
        pan = {"v0": v0, "v1": v1, "vn": vn, "vnp": vnp}
        out = []
        for r in rows:
            acc = np.zeros(self.width, dtype=complex)
            for slot in SLOTS:
                if pan[slot] is not None:
                    blk = self.G[(r, slot)]
                    if self.counter is not None:
                        self.counter[0] += blk.shape[0] * blk.shape[1]
                    acc += blk @ pan[slot]
            out.append(acc)
        return out


class InnerLU:
    """Unpivoted block-tridiagonal LU of the assembled cell-interface system (``nested.py:156-254``):
    2w x 2w blocks per interface from the cells' Green blocks, pivot blocks inverted, both substitutions
    as matrix-vector products; every matvec counts rows x cols touches (``nested.py:67-73``)."""

    def __init__(self, cells, counter):
        self.counter = counter
        nI = len(cells) - 1
        self.nI = nI
        w = cells[0].width
        self.w = w
        eye = np.eye(w, dtype=complex)
        zero = np.zeros((w, w), dtype=complex)
        self.diag, self.lower, self.upper = [], [None], []
        for i in range(nI):
            gi, gp, n_i = cells[i].G, cells[i + 1].G, cells[i].n
            self.diag.append(np.block([[eye - gi[(n_i, "vn")], -gi[(n_i, "vnp")]],
                                       [-gp[(1, "v0")], eye - gp[(1, "v1")]]]))
            if i >= 1:
                self.lower.append(np.block([[-gi[(n_i, "v0")], -gi[(n_i, "v1")]], [zero, zero]]))
            self.upper.append(np.block([[zero, zero], [-gp[(1, "vn")], -gp[(1, "vnp")]]])
                              if i <= nI - 2 else None)
        self.pivinv = []
        for i in range(nI):
            piv = self.diag[i].copy()
            if i >= 1:
                piv -= self.lower[i] @ (self.pivinv[i - 1] @ self.upper[i - 1])
            self.pivinv.append(np.linalg.inv(piv))

    def _mv(self, mat, v):
        self.counter[0] += mat.shape[0] * mat.shape[1]
        return mat @ v

    def solve(self, b):
        y = [b[0]]
        for i in range(1, self.nI):
            y.append(b[i] - self._mv(self.lower[i], self._mv(self.pivinv[i - 1], y[i - 1])))
        x = [None] * self.nI
        x[-1] = self._mv(self.pivinv[-1], y[-1])
        for i in range(self.nI - 2, -1, -1):
            x[i] = self._mv(self.pivinv[i], y[i] - self._mv(self.upper[i], x[i + 1]))
        return x


class NestedLayer:
    """One layer solved by the swapped cell decomposition (``nested.py:272-353``).

    ``boundary_samples``/``newton_samples``/``add_sources`` mirror
    ``LayerOperator`` (``subdomain.py:157-199``); ``solve`` is Alg. 7:
    swap, split, cell Newton tables, inner polarized-traces GMRES
    (``nested.py:125-153``), per-cell reconstruction, swap back.
    """

    def __init__(self, nx, n, h, npml, c_layer, C, omega, Lc, inner_ktol=1e-6,
                 inner_max_iter=200, backend="pt"):
        self.nx, self.n, self.h, self.npml = nx, n, h, npml
        self.wx, self.wz = nx + 2 * npml, n + 2 * npml
        self.width = self.wx
        self.shape = (self.wz, self.wx)
        self.inner_ktol, self.inner_max_iter = inner_ktol, inner_max_iter
        self.counter = [0]
        self.inner_iters = []
        # the layer's own operator is only needed for its cut blocks (subdomain.py:129)
        self.H = fd_operator(nx, n, h, npml, c_layer, C, omega)
        self._blk = {}
        cext = split_extents(nx, Lc)  # partition_layers(sgrid, Lc), nested.py:294-296
        self.cell_offsets = _offsets(cext)
        cT = np.asarray(c_layer).T  # model.transposed()
        self.cells = []
        for ci, nxc in enumerate(cext):
            off = self.cell_offsets[ci]
            ccell = cT[off : off + nxc + 2 * npml, :]
            self.cells.append(Cell(n, nxc, h, npml, ccell, C, omega, counter=self.counter))
        self.inner = Traces(self.cells, self.cell_offsets)
        self.backend = backend
        self.lu = InnerLU(self.cells, self.counter) if backend == "lu" and Lc > 1 else None

    row = Local.row
    block = Local.block
    add_sources = Local.add_sources

    def solve(self, rhs):  # nested.py:344-353
        g = np.asarray(rhs, dtype=complex).reshape(self.shape).T.copy()
        fc = self.inner.split(g)
        if self.inner.nI == 0:
            t = np.zeros((0, 2, self.inner.w), dtype=complex)
        elif self.lu is not None:  # nested.py:322-342 with _InnerLU: rows n of cell i and 1 of cell i+1
            d, p = self.inner.newton_rhs(fc)
            x = self.lu.solve([np.concatenate([-d[i, 0], -p[i, 1]]) for i in range(self.inner.nI)])
            w = self.inner.w
            t = np.zeros((self.inner.nI, 2, w), dtype=complex)
            for i in range(self.inner.nI):
                t[i, 0] = x[i][:w]
                t[i, 1] = x[i][w:]
        else:
            d, p = self.inner.newton_rhs(fc)
            op, pre, unpack = self.inner.flat_ops("gs")
            x, its, hist, ok = gmres(op, np.concatenate([d.ravel(), p.ravel()]), pre,
                                     self.inner_ktol, self.inner_max_iter)
            self.inner_iters.append(its)
            if not ok:
                raise InnerSolveError(f"inner trace solve stalled at {hist[-1]:.3e}")
            a, b = unpack(x)
            t = a + b
        v = self.inner.reconstruct(t, fc, g.shape)
        return v.T.copy()

    def boundary_samples(self, v0, v1, vn, vnp, rows):
        rhs = self.add_sources(np.zeros(self.shape, dtype=complex), v0, v1, vn, vnp)
        w = self.solve(rhs)
        return [w[self.row(r)].copy() for r in rows]

    def newton_samples(self, f, rows):
        w = self.solve(f)
        return [w[self.row(r)].copy() for r in rows]


# --------------------------------------------------------------------------
# outer solve (sie.py:361-445, nested.py:507-521)


@dataclass
class OracleResult:
    u: np.ndarray
    iterations: float
    residuals: list = field(default_factory=list)
    converged: bool = True
    relative_residual: float = 0.0
    traces: np.ndarray | None = None
    touches: int = 0
    inner_iterations: list = field(default_factory=list)


class OracleSolver:
    """``build_nested_layers(..., backend="pt")`` + ``PolarizedTracesSolver``.

    ``nested=False`` gives the direct-layer solver (``LayerWorkspace``
    layers, ``sie.py:375-379``) used by the reference's own end-to-end tests.
    """

    def __init__(self, nx, nz, h, npml, c, C, omega, extents, Lc=1, nested=True,
                 inner_ktol=1e-6, inner_max_iter=200, backend="pt"):
        self.nx, self.nz, self.h, self.npml = nx, nz, h, npml
        self.shape = (nz + 2 * npml, nx + 2 * npml)
        self.c = np.asarray(c, dtype=float)
        self.C, self.omega = C, omega
        self.extents = tuple(extents)
        offs = _offsets(self.extents)
        layers = []
        for ell, n in enumerate(self.extents):
            off = offs[ell]
            cl = self.c[off : off + n + 2 * npml, :]
            if nested:
                layers.append(NestedLayer(nx, n, h, npml, cl, C, omega, Lc, inner_ktol,
                                          inner_max_iter, backend))
            else:
                layers.append(Local(nx, n, h, npml, cl, C, omega))
        self.outer = Traces(layers, offs)
        self._H = None

    @classmethod
    def from_problem(cls, prob, nested=True, **kw):
        g = prob.grid
        return cls(g.nx, g.nz, g.h, g.npml, prob.model.c, prob.pml.C, prob.pml.omega,
                   prob.partition.extents, prob.Lc, nested=nested,
                   inner_ktol=kw.get("inner_ktol", prob.inner_ktol), backend=kw.get("backend", "pt"),
                   inner_max_iter=kw.get("inner_max_iter", 200))

    def global_operator(self):
        if self._H is None:
            self._H = fd_operator(self.nx, self.nz, self.h, self.npml, self.c, self.C,
                                  self.omega)
        return self._H

    def touches(self):
        return int(sum(getattr(s, "counter", [0])[0] for s in self.outer.slabs))

    def solve(self, f, ktol=1e-7, max_iter=200, restart=0, preconditioner="gs", method="gmres"):
        """``PolarizedTracesSolver.solve`` (sie.py:392-439); ``method`` as ``KrylovConfig.method``
        (``krylov.py:204-214``)."""
        f = np.asarray(f, dtype=complex).reshape(self.shape)
        T = self.outer
        for s in T.slabs:
            if hasattr(s, "counter"):
                s.counter[0] = 0
                s.inner_iters = []
        fl = T.split(f)
        if np.linalg.norm(f) == 0.0:
            return OracleResult(np.zeros(self.shape, dtype=complex), 0.0, [0.0])
        if T.nI == 0:
            u = T.reconstruct(np.zeros((0, 2, T.w), dtype=complex), fl, self.shape)
            r = self._relres(u, f)
            return OracleResult(u, 0.0, [r], True, r)
        d, p = T.newton_rhs(fl)
        op, pre, unpack = T.flat_ops(preconditioner)
        if method == "bicgstab":
            x, its, hist, ok = bicgstab(op, np.concatenate([d.ravel(), p.ravel()]), pre, ktol, max_iter)
        else:
            x, its, hist, ok = gmres(op, np.concatenate([d.ravel(), p.ravel()]), pre, ktol,
                                     max_iter, restart)
        if not ok:
            raise KrylovBreakdown(f"trace solve did not reach {ktol:g}", residuals=hist)
        a, b = unpack(x)
        t = a + b
        u = T.reconstruct(t, fl, self.shape)
        inner = [list(s.inner_iters) for s in T.slabs if hasattr(s, "inner_iters")]
        return OracleResult(u, its, hist, ok, self._relres(u, f), t, self.touches(), inner)

    def _relres(self, u, f):  # sie.py:441-445
        H = self.global_operator()
        return float(np.linalg.norm(H @ u.ravel() - f.ravel()) / np.linalg.norm(f))
