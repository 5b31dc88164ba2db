"""Host-side problem description: grids, PML ramps, media, partitions, sources.

These are the value types the reference's construction API takes
(``Grid``/``PmlProfile``/``VelocityModel`` in
``/root/reference/pkg/src/polartraces/discretization.py:58-220``,
``LayerPartition``/``partition_layers`` in ``subdomain.py:51-110``).  They are
re-stated here so the B200 package is a drop-in on a box where the reference is
not installed.  Nothing in this module runs in the online stage: it feeds the
offline coefficient builder (``offline.py``), whose output is uploaded once.

Conventions (identical to the reference):

* extended array ``(wz, wx) = (nz + 2 npml, nx + 2 npml)``, depth-major, C order;
  lattice depth ``q`` lives in array row ``q + npml - 1`` (``discretization.py:115-120``);
* the 5-point operator is ``kron(I_z, T_x) + kron(T_z, I_x) - omega^2 diag(1/c^2)``
  (``discretization.py:223-251``) where each ``T`` is the PML-stretched
  second difference; only its three diagonals are ever formed here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "Grid",
    "PmlProfile",
    "VelocityModel",
    "DiscretizationSpec",
    "LayerPartition",
    "CellPartition",
    "default_pml_strength",
    "default_npml",
    "partition_layers",
    "partition_cells",
    "delta_source",
    "axis_tridiag",
]

_PML_ATTENUATION = 1e-6


def default_pml_strength(c_ref):
    """``1.5 ln(1e6) c_ref`` -- ``discretization.py:48-50``."""
    return 1.5 * np.log(1.0 / _PML_ATTENUATION) * c_ref


def default_npml(nx, nz):
    """``max(10, ceil(log2(nx nz)))`` -- ``discretization.py:53-55``."""
    return max(10, int(np.ceil(np.log2(nx * nz))))


@dataclass(frozen=True)
class Grid:
    """Tensor grid of one (sub)domain -- ``discretization.py:58-123``."""

    nx: int
    nz: int
    h: float
    npml: int
    origin: tuple = (0, 0)

    def __post_init__(self):
        if self.nx < 1 or self.nz < 1:
            raise ValueError("grid needs nx, nz >= 1")
        if self.h <= 0:
            raise ValueError("grid spacing must be positive")
        if self.npml < 0:
            raise ValueError("npml must be nonnegative")

    @property
    def wx(self):
        return self.nx + 2 * self.npml

    @property
    def wz(self):
        return self.nz + 2 * self.npml

    @property
    def shape(self):
        return (self.wz, self.wx)

    @property
    def n_unknowns(self):
        return self.wx * self.wz

    @property
    def lx(self):
        return (self.nx + 1) * self.h

    @property
    def lz(self):
        return (self.nz + 1) * self.h

    def x_coords(self):
        return self.h * np.arange(1 - self.npml, self.nx + self.npml + 1, dtype=float)

    def z_coords(self):
        return self.h * np.arange(1 - self.npml, self.nz + self.npml + 1, dtype=float)

    def row_of(self, q):
        return q + self.npml - 1

    def col_of(self, p):
        return p + self.npml - 1

    def transposed(self):
        return Grid(self.nz, self.nx, self.h, self.npml, (self.origin[1], self.origin[0]))


@dataclass(frozen=True)
class PmlProfile:
    """Quadratic absorbing ramps -- ``discretization.py:126-176``.

    ``sigma(s) = C/delta ((s - edge)/delta)^2`` outside ``[0, span]``,
    ``alpha = 1/(1 + i sigma/omega)``, ``delta = npml h``.
    """

    npml: int
    h: float
    C: float
    omega: float

    def __post_init__(self):
        if self.C <= 0:
            raise ValueError("absorption strength C must be positive")
        if self.omega <= 0:
            raise ValueError("omega must be positive")

    @property
    def delta(self):
        return self.npml * self.h

    def sigma(self, s, span):
        s = np.asarray(s, dtype=float)
        out = np.zeros_like(s)
        if self.npml == 0:
            return out
        d = self.delta
        lo = s < 0.0
        hi = s > span
        out[lo] = (self.C / d) * (s[lo] / d) ** 2
        out[hi] = (self.C / d) * ((s[hi] - span) / d) ** 2
        return out

    def alpha(self, sigma):
        return 1.0 / (1.0 + 1j * np.asarray(sigma) / self.omega)

    def alpha_axis(self, n, half=0.0):
        """alpha at the extended nodes of an n-point axis, shifted by ``half`` h."""
        coords = self.h * (np.arange(1 - self.npml, n + self.npml + 1, dtype=float) + half)
        return self.alpha(self.sigma(coords, (n + 1) * self.h))


class VelocityModel:
    """Wave speed on the extended nodes -- ``discretization.py:193-220``."""

    def __init__(self, grid, c):
        c = np.asarray(c, dtype=float)
        if c.shape != grid.shape:
            raise ValueError(f"model shape {c.shape} does not match extended grid {grid.shape}")
        if not np.all(np.isfinite(c)) or np.any(c <= 0):
            raise ValueError("wave speeds must be positive and finite")
        self.grid = grid
        self.c = c

    @property
    def m(self):
        return 1.0 / self.c**2

    @classmethod
    def constant(cls, grid, c0=1.0):
        return cls(grid, np.full(grid.shape, float(c0)))

    def restrict(self, grid, row0, col0):
        return VelocityModel(grid, self.c[row0 : row0 + grid.wz, col0 : col0 + grid.wx].copy())

    def transposed(self):
        return VelocityModel(self.grid.transposed(), self.c.T.copy())


@dataclass(frozen=True)
class DiscretizationSpec:
    """Volume discretization selector -- ``subdomain.py:35-48``.

    Only the 5-point finite-difference operator (``kind="fd"``, the one every
    benchmark config uses) has a B200 online path; Q1 is out of scope
     and is rejected at construction.
    """

    kind: str = "fd"
    smoothness_threshold: float = 1.05
    quad_tol: float = 1e-8

    def __post_init__(self):
        if self.kind not in ("fd", "q1"):
            raise ValueError(f"unknown discretization {self.kind!r}")


def axis_tridiag(pml, n, h):
    """Three diagonals of the PML-stretched 1-D second difference ``T``.

    Follows ``assemble_fd.axis_tridiag`` (``discretization.py:237-244``):
    ``main = a0 (a+ + a-)/h^2``, ``upper[i] = -a0[i] a+[i]/h^2`` (i < N-1),
    ``lower[i] = -a0[i] a-[i]/h^2`` (i >= 1).  Returned as three length-N
    arrays with ``lower[0] = upper[N-1] = 0``.
    """
    a0 = pml.alpha_axis(n, 0.0)
    ap = pml.alpha_axis(n, +0.5)
    am = pml.alpha_axis(n, -0.5)
    h2 = h * h
    main = a0 * (ap + am) / h2
    upper = -(a0 * ap / h2)
    lower = -(a0 * am / h2)
    upper[-1] = 0.0
    lower[0] = 0.0
    return lower, main, upper


@dataclass(frozen=True)
class LayerPartition:
    """Depth extents of each layer -- ``subdomain.py:51-73``."""

    extents: tuple

    @property
    def L(self):
        return len(self.extents)

    @property
    def offsets(self):
        return tuple(int(v) for v in np.concatenate([[0], np.cumsum(self.extents)[:-1]]))

    @property
    def n_interfaces(self):
        return self.L - 1

    def interface_rows(self):
        return tuple(int(v) for v in np.cumsum(self.extents)[:-1])


@dataclass(frozen=True)
class CellPartition:
    extents: tuple
    swapped: bool = True

    @property
    def Lc(self):
        return len(self.extents)


def _split(n, parts):
    base, rem = divmod(n, parts)
    return tuple(base + 1 if i < rem else base for i in range(parts))


def partition_layers(grid, L):
    """Near-equal slabs, remainder on top -- ``subdomain.py:88-100``."""
    nz = grid.nz if isinstance(grid, Grid) else int(grid)
    if L < 1:
        raise ValueError("need at least one layer")
    if nz < 2 * L:
        raise ValueError(f"{L} layers need nz >= {2 * L}, got {nz}")
    return LayerPartition(_split(nz, L))


def partition_cells(grid, Lc):
    """``subdomain.py:103-110``."""
    nx = grid.nx if isinstance(grid, Grid) else int(grid)
    if Lc < 1:
        raise ValueError("need at least one cell")
    if Lc > 1 and nx < 2 * Lc:
        raise ValueError(f"{Lc} cells need nx >= {2 * Lc}, got {nx}")
    return CellPartition(_split(nx, Lc))


def assemble_fd(grid, model, pml):
    """The global 5-point operator ``-Delta_PML - omega^2 m`` on the extended grid (``discretization.py:223-251``
    of the reference): ``kron(I_z, T_x) + kron(T_z, I_x) - omega^2 diag(1/c^2)``, depth-major unknowns, as a
    scipy CSR matrix.  The device path never forms it; this backs ``PolarizedTracesSolver.global_operator()``."""
    import scipy.sparse as sp

    def axis(n):
        lower, main, upper = axis_tridiag(pml, n, grid.h)
        return sp.diags([lower[1:], main, upper[:-1]], [-1, 0, 1], format="csr")

    Tx, Tz = axis(grid.nx), axis(grid.nz)
    m = 1.0 / np.asarray(model.c, dtype=float) ** 2
    return (sp.kron(sp.eye(grid.wz), Tx) + sp.kron(Tz, sp.eye(grid.wx))
            - pml.omega ** 2 * sp.diags(m.ravel())).tocsr().astype(np.complex128)


def delta_source(grid, node, discretization="fd"):
    """Discrete point source ``1/h^2`` at lattice node (p, q) -- ``discretization.py:456-471``."""
    p, q = node
    if not (1 - grid.npml <= p <= grid.nx + grid.npml) or not (
        1 - grid.npml <= q <= grid.nz + grid.npml
    ):
        raise ValueError(f"node {node} outside the extended grid")
    out = np.zeros(grid.shape, dtype=complex)
    out[grid.row_of(q), grid.col_of(p)] = 1.0 / grid.h**2 if discretization == "fd" else 1.0
    return out
