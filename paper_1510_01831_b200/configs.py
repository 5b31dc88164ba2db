"""The five synthetic benchmark media of BASELINE.json, as one shared generator.

Both the B200 path and the CPU oracle build their inputs from here, so the two
sides solve identical problems.  The conventions are the ones pinned in
SURVEY.md section 8(d):

* ``h = 1/(nz+1)`` (unit depth); the medium is evaluated at the extended node
  coordinates (``Grid.x_coords``/``z_coords``); noise lives on the extended array;
* ``C = default_pml_strength(max c)``;
* point sources ``delta_source(grid, (round(x/h), round(z/h)))``; equispaced
  surface sources ``p_i = round((i+1)(nx+1)/(n_src+1))``, ``q = 1``;
* every random draw comes from ``np.random.default_rng(0)``;
* ``KrylovConfig(ktol=1e-9, max_iter=200)``, GS preconditioner, ``inner_ktol=1e-6``.

The BP2004/Marmousi2 models of the paper are not used (not available); these
seeded media stand in for them.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .discretization import (
    Grid,
    PmlProfile,
    VelocityModel,
    default_pml_strength,
    delta_source,
    partition_layers,
)

__all__ = ["Problem", "make_config", "CONFIG_NAMES", "small_problem"]

CONFIG_NAMES = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")


@dataclass
class Problem:
    name: str
    grid: Grid
    model: VelocityModel
    pml: PmlProfile
    partition: object
    Lc: int
    sources: list  # lattice nodes (p, q)
    ktol: float = 1e-9
    max_iter: int = 200
    inner_ktol: float = 1e-6
    notes: dict = field(default_factory=dict)

    def rhs(self, idx=None):
        """Point-source right-hand sides, shape (nsrc, wz, wx) complex128."""
        nodes = self.sources if idx is None else [self.sources[i] for i in idx]
        return np.stack([delta_source(self.grid, nd) for nd in nodes])

    @property
    def unknowns(self):
        return self.grid.nx * self.grid.nz


def _smooth_noise(rng, shape, corr):
    """White noise smoothed by a Gaussian of ``corr`` grid points, unit std."""
    from scipy.ndimage import gaussian_filter

    w = rng.standard_normal(shape)
    s = gaussian_filter(w, sigma=corr, mode="reflect")
    return s / s.std()


def _layered(grid, rng, n_strata=12, vmin=1.5, vmax=4.5, jitter=0.3, dip_deg=15.0,
             noise=0.05, corr=10.0):
    x = grid.x_coords()
    z = grid.z_coords()
    X, Z = np.meshgrid(x, z)  # depth-major (wz, wx)
    lx, lz = grid.lx, grid.lz
    depths = np.sort(rng.uniform(0.05 * lz, 0.95 * lz, n_strata - 1))
    dips = np.deg2rad(rng.uniform(-dip_deg, dip_deg, n_strata - 1))
    vel = np.linspace(vmin, vmax, n_strata) + rng.uniform(-jitter, jitter, n_strata)
    idx = np.zeros(grid.shape, dtype=int)
    for d, a in zip(depths, dips):
        idx += (Z > d + np.tan(a) * (X - 0.5 * lx)).astype(int)
    c = vel[idx]
    c = c * (1.0 + noise * _smooth_noise(rng, grid.shape, corr))
    return c


def _points_in_polygon(px, pz, poly):
    """Even-odd rule point-in-polygon on arrays (no matplotlib dependency)."""
    inside = np.zeros(px.shape, dtype=bool)
    n = len(poly)
    for i in range(n):
        x1, z1 = poly[i]
        x2, z2 = poly[(i + 1) % n]
        cond = (z1 > pz) != (z2 > pz)
        with np.errstate(divide="ignore", invalid="ignore"):
            xint = (x2 - x1) * (pz - z1) / (z2 - z1) + x1
        inside ^= cond & (px < xint)
    return inside


def _salt_model(grid, rng, noise=0.05, corr=10.0):
    x = grid.x_coords()
    z = grid.z_coords()
    X, Z = np.meshgrid(x, z)
    lx, lz = grid.lx, grid.lz
    c = 1.5 + 2.0 * np.clip(Z, 0.0, lz) / lz
    c = c * (1.0 + noise * _smooth_noise(rng, grid.shape, corr))
    nv = 24
    ang = np.linspace(0.0, 2 * np.pi, nv, endpoint=False)
    rad = 0.15 * lx * (1.0 + rng.uniform(-0.3, 0.3, nv))
    cx, cz = 0.5 * lx, 0.45 * lz
    poly = np.stack([cx + rad * np.cos(ang), cz + rad * np.sin(ang)], axis=1)
    c[_points_in_polygon(X, Z, poly)] = 4.5
    return c


def _surface_sources(grid, n_src, q=1):
    return [(int(round((i + 1) * (grid.nx + 1) / (n_src + 1))), q) for i in range(n_src)]


def make_config(name, n_sources=None):
    """Build one of the BASELINE.json configs (``cfg1`` .. ``cfg5``)."""
    rng = np.random.default_rng(0)
    if name == "cfg1":
        nx = nz = 160
        npml = 10
        h = 1.0 / (nz + 1)
        grid = Grid(nx, nz, h, npml)
        model = VelocityModel.constant(grid, 1.0)
        omega = 2 * np.pi * 16
        L, Lc = 4, 2
        sources = [(int(round(0.5 / h)), int(round(0.25 / h)))]
    elif name == "cfg2":
        nx = nz = 400
        npml = 10
        h = 1.0 / (nz + 1)
        grid = Grid(nx, nz, h, npml)
        X, Z = np.meshgrid(grid.x_coords(), grid.z_coords())
        c = 1.0 - 0.4 * np.exp(-((X - 0.5) ** 2 + (Z - 0.5) ** 2) / 0.02)
        model = VelocityModel(grid, c)
        omega = 2 * np.pi * 0.6 / (8 * h)
        L, Lc = 8, 4
        xs = rng.uniform(0.1, 0.9, 16)
        sources = [(int(round(x / h)), int(round(0.1 / h))) for x in xs]
    elif name == "cfg3":
        nx = nz = 1000
        npml = 12
        h = 1.0 / (nz + 1)
        grid = Grid(nx, nz, h, npml)
        model = VelocityModel(grid, _layered(grid, rng))
        omega = 2 * np.pi * 1.5 / (8 * h)
        L, Lc = 16, 8
        sources = _surface_sources(grid, 64, q=int(round(0.02 / h)))
    elif name == "cfg4":
        nx, nz = 2000, 1000
        npml = 12
        h = 1.0 / (nz + 1)
        grid = Grid(nx, nz, h, npml)
        model = VelocityModel(grid, _salt_model(grid, rng))
        omega = 2 * np.pi * 1.5 / (10 * h)
        L, Lc = 20, 16
        sources = _surface_sources(grid, 256)
    elif name == "cfg5":
        nx = nz = 3000
        npml = 16
        h = 1.0 / (nz + 1)
        grid = Grid(nx, nz, h, npml)
        model = VelocityModel(grid, _layered(grid, rng))
        omega = 2 * np.pi * 1.5 / (8 * h)
        L, Lc = 32, 16
        sources = _surface_sources(grid, 64)
    else:
        raise ValueError(f"unknown config {name!r}")
    pml = PmlProfile(npml, h, default_pml_strength(float(model.c.max())), omega)
    part = partition_layers(grid, L)
    if n_sources is not None:
        sources = sources[:n_sources]
    return Problem(name, grid, model, pml, part, Lc, sources)


def small_problem(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0, contrast=0.4, seed=0,
                  n_sources=2):
    """Seeded random-medium toy problem in the style of the reference tests
    (``test_sie.py:21-30``): ``c = 1 + contrast * U[0,1)``."""
    h = 1.0 / (nx + 1)
    grid = Grid(nx, nz, h, npml)
    rng = np.random.default_rng(seed)
    c = 1.0 + contrast * rng.random(grid.shape)
    model = VelocityModel(grid, c)
    pml = PmlProfile(npml, h, default_pml_strength(1.0 + contrast), omega)
    part = partition_layers(grid, L)
    srcs = [(int(p), int(q)) for p, q in zip(rng.integers(1, nx + 1, n_sources),
                                             rng.integers(1, nz + 1, n_sources))]
    return Problem(f"small{nx}x{nz}L{L}c{Lc}", grid, model, pml, part, Lc, srcs)
