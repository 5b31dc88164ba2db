"""Drop-in construction and ``solve()`` API of the reference, running on one B200.

Mirrors the reference's user-facing path

    layers = build_nested_layers(grid, model, pml, partition, Lc=Lc, backend="pt")
    solver = PolarizedTracesSolver(grid, model, pml, partition, layers=layers)
    res = solver.solve(f, KrylovConfig(ktol=1e-9))

(``nested.py:507-521``, ``sie.py:361-445``) with identical argument meaning,
return type (``SolveResult``) and exceptions (``KrylovBreakdown``,
``InnerSolveError``, ``ValueError``).  Construction runs the offline stage
(``offline.py``) and uploads it once (``pt_create``); ``solve`` is one call
into the C ABI (``pt_solve``), which runs the whole online stage -- Newton
tables, outer GMRES with its layer-solves, inner polarized-traces GMRES, cell
solves and reconstruction -- on the device.  ``solve_many`` solves a batch of
sources in lockstep (the reference loops ``solve``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .discretization import DiscretizationSpec, Grid
from .krylov import InnerSolveError, KrylovBreakdown, KrylovConfig
from .offline import build_factors, residual_from_operator

__all__ = [
    "TraceStack",
    "PolarizedTraceStack",
    "SolveResult",
    "NestedLayers",
    "build_nested_layers",
    "PolarizedTracesSolver",
]


class TraceStack:
    """(interfaces, 2, width) panels -- ``sie.py:37-77``."""

    __slots__ = ("data",)

    def __init__(self, data):
        self.data = np.asarray(data, dtype=complex)

    @classmethod
    def zeros(cls, n_interfaces, width):
        return cls(np.zeros((n_interfaces, 2, width), dtype=complex))

    @property
    def n_interfaces(self):
        return self.data.shape[0]

    @property
    def width(self):
        return self.data.shape[2]

    def flat(self):
        return self.data.ravel().copy()

    def copy(self):
        return TraceStack(self.data.copy())

    def norm(self):
        return np.linalg.norm(self.data)

    def __add__(self, other):
        return TraceStack(self.data + other.data)

    def __sub__(self, other):
        return TraceStack(self.data - other.data)

    def __getitem__(self, idx):
        return self.data[idx]


class PolarizedTraceStack:
    """Down/up stacks -- ``sie.py:80-109``."""

    __slots__ = ("down", "up")

    def __init__(self, down, up):
        self.down = down
        self.up = up

    @classmethod
    def from_flat(cls, flat, n_interfaces, width):
        flat = np.asarray(flat, dtype=complex)
        half = flat.size // 2
        return cls(TraceStack(flat[:half].reshape(n_interfaces, 2, width)),
                   TraceStack(flat[half:].reshape(n_interfaces, 2, width)))

    def flat(self):
        return np.concatenate([self.down.flat(), self.up.flat()])

    def reassemble(self):
        return self.down + self.up


@dataclass
class SolveResult:
    """``sie.py:349-358``."""

    u: np.ndarray
    iterations: float
    residuals: list = field(default_factory=list)
    converged: bool = True
    relative_residual: float = 0.0
    kappa_margin: float = 0.0
    traces: TraceStack | None = None
    polarized: PolarizedTraceStack | None = None


class NestedLayers(list):
    """What ``build_nested_layers`` returns: one entry per layer plus the offline
    factors of the whole partition (the device upload happens in the solver)."""

    def __init__(self, items, factors, Lc, backend, inner_ktol, inner_max_iter):
        super().__init__(items)
        self.factors = factors
        self.Lc = Lc
        self.backend = backend
        self.inner_ktol = inner_ktol
        self.inner_max_iter = inner_max_iter


@dataclass
class LayerDescriptor:
    index: int
    n: int
    width: int
    grid: Grid
    Lc: int


def is_reference_layers(layers):
    """The reference's own layer objects: ``NestedLayerSolver`` (``nested.py:272``, has ``cells`` and
    ``blocksets``) or direct ``LayerWorkspace`` layers (``subdomain.py:202``, has ``lu`` and ``H``)."""
    if isinstance(layers, NestedLayers) or not layers:
        return False
    first = layers[0]
    return (hasattr(first, "cells") and hasattr(first, "blocksets")) or (hasattr(first, "lu") and hasattr(first, "H"))


def from_reference_layers(layers, grid, model, pml, partition, device=None, inner_dense=None):
    """``NestedLayers`` for this path from the reference's own offline objects: the list
    ``build_nested_layers(...)`` of the reference returns (``nested.py:507-521``), or its direct layers
    (``build_layer``, ``subdomain.py:227-236``).  The cell couplings are read from the reference's assembled
    operators and its ``GreenBlockSet`` matrices are uploaded as they are (``offline.build_factors``,
    ``reference_layers=``); the inner solver settings (backend, ``inner_ktol``, ``inner_max_iter``,
    ``assembled_boundary``) are the layers' own."""
    first = layers[0]
    if hasattr(first, "cells"):
        Lc = len(first.cells)
        backend = first.backend
        inner_ktol = first.inner_ktol
        inner_max_iter = getattr(getattr(first, "inner", None), "max_iter", 200)
        assembled = bool(getattr(first, "assembled_boundary", False))
        # PLR-compressed Green blocks (plr.py:96-219, green.py:124-126): the reference's GreenBlockSet.dense()
        # expands them (as its own artifact dump does, green.py:156-163); the device applies the expanded block
        # (U V) x where the reference applies U (V x) -- the same linear map.  TouchCounter totals then count
        # dense touches, not the PLR leaves'.
    else:
        Lc, backend, inner_ktol, inner_max_iter, assembled = 1, "pt", 1e-6, 200, False
    if len(layers) != partition.L:
        raise ValueError(f"{len(layers)} layers for a partition of {partition.L}")
    return build_nested_layers(grid, model, pml, partition, Lc=Lc, backend=backend, inner_ktol=inner_ktol,
                               inner_max_iter=inner_max_iter, assembled_boundary=assembled, device=device,
                               inner_dense=inner_dense, reference_layers=list(layers))


def build_nested_layers(grid, model, pml, partition, disc=DiscretizationSpec(), Lc=1, backend="pt",
                        inner_ktol=1e-6, inner_max_iter=200, plr_threshold=None, plr_eps=1e-8,
                        plr_max_rank=None, seed=0, assembled_boundary=False, device=None, inner_dense=None,
                        reference_layers=None, cell_solver=None, **unused):
    """``nested.py:507-521`` (with ``NestedLayerSolver`` kwargs, ``nested.py:279-281``).

    Runs the offline stage (Schur factors + Green blocks) for every layer.
    ``device`` selects where the offline arithmetic runs: a CUDA device (the
    default when one is present; the unit-source cell solves then run on the
    K1 kernel, ``cell_solver="k1"``) or ``"cpu"`` (torch on the host, small
    problems and CPU-only tests); its output is uploaded by the solver.
    ``inner_dense`` (None = by Lc) builds the dense inner operators that let
    the inner GMRES run as one dense product per step.
    """
    if backend not in ("pt", "lu"):
        raise ValueError(f"unknown inner backend {backend!r}")  # nested.py:283-284
    if disc.kind != "fd":
        raise NotImplementedError("only the finite-difference discretization has a B200 path")
    if plr_threshold is not None:
        raise NotImplementedError("PLR compression is not part of the B200 path (off in every config)")
    if Lc < 1:
        raise ValueError("need at least one cell")
    if Lc > 1 and grid.nx < 2 * Lc:
        raise ValueError(f"{Lc} cells need nx >= {2 * Lc}, got {grid.nx}")
    if device is None:
        import torch

        device = f"cuda:{torch.cuda.current_device()}" if torch.cuda.is_available() else "cpu"
    F = build_factors(grid, model, pml, partition, Lc, device=device, inner_dense=inner_dense,
                      backend=backend, reference_layers=reference_layers, cell_solver=cell_solver)
    # assembled_boundary (nested.py:355-486): boundary samples through M_f -> inner solve -> direct + M_u.
    # This path's sample-only layer solves already are those linear maps (pass-0 operator = M_f and the
    # direct part, sampled trace response = M_u); the flag selects the reference's touch accounting.
    F.assembled_boundary = bool(assembled_boundary) and Lc > 1
    items = []
    for ell, (n, off) in enumerate(zip(partition.extents, partition.offsets)):
        lgrid = Grid(grid.nx, n, grid.h, grid.npml, origin=(grid.origin[0], grid.origin[1] + off))
        items.append(LayerDescriptor(ell, n, grid.wx, lgrid, Lc))
    return NestedLayers(items, F, Lc, backend, inner_ktol, inner_max_iter)


_ERR = {
    _abi.PT_INNER_NOT_CONVERGED: InnerSolveError,
    _abi.PT_BREAKDOWN: KrylovBreakdown,
    _abi.PT_BAD_ARGUMENT: ValueError,
}


class PolarizedTracesSolver:
    """``sie.py:361-445`` on the B200 online path.

    ``layers=None`` gives direct (unsplit) layer solves like the reference's
    ``LayerWorkspace`` layers; on this path that is the one-cell
    decomposition (Lc = 1), i.e. one exact block-tridiagonal solve per layer.
    """

    def __init__(self, grid, model, pml, partition, disc=DiscretizationSpec(), layers=None,
                 global_operator=None, device=0):
        self.grid = grid
        self.model = model
        self.pml = pml
        self.partition = partition
        self.disc = disc
        if layers is None:
            layers = build_nested_layers(grid, model, pml, partition, disc, Lc=1)
        elif is_reference_layers(layers):  # the reference's own build_nested_layers / build_layer output
            layers = from_reference_layers(layers, grid, model, pml, partition)
        if not isinstance(layers, NestedLayers):
            raise TypeError("layers must come from build_nested_layers (this package's or the reference's)")
        self.layers = layers
        self.nI = partition.L - 1
        self._H = global_operator
        F = layers.factors
        if global_operator is not None:  # the true residual uses the caller's operator (sie.py:381, 441-445)
            F.tx, F.tz, F.hdiag = residual_from_operator(global_operator, F.wz, F.wx)
        self.ctx = _abi.Context(F, device=device)

    def global_operator(self):
        """``sie.py:387-390``: the caller's operator, or the FD operator of (grid, model, pml) assembled lazily."""
        if self._H is None:
            from .discretization import assemble_fd

            self._H = assemble_fd(self.grid, self.model, self.pml)
        return self._H

    def close(self):
        self.ctx.close()

    def release_offline_arrays(self):
        """Drop this object's references to the offline arrays once ``pt_create`` has copied them to the device:
        when the offline stage ran on the GPU (``build_nested_layers(device="cuda")``) this frees a full second
        copy of the factors in HBM (tens of GB for cfg5).  Geometry and scalars stay available."""
        F = self.layers.factors
        for lf in F.layers:
            lf.dense = lf.lu_inv = None
            for cf in lf.cells:
                cf.sinv = cf.green = cf.gsmp = cf.q0 = None
        self.ctx.keep = None

    # -- one call into the C ABI for a batch of sources
    def _run(self, F, config, preconditioner, device_arrays=None, out=None):
        if preconditioner not in ("gs", "jac"):
            raise ValueError(f"unknown preconditioner {preconditioner!r}")
        R = F.shape[0] if device_arrays is None else device_arrays[2]
        cfg = _abi.PtKrylov(config.ktol, config.max_iter, config.restart, self.layers.inner_ktol,
                            self.layers.inner_max_iter, 0 if preconditioner == "gs" else 1,
                            0 if config.method == "gmres" else 1)
        L_ = _abi.lib()
        wz, wx = self.grid.shape
        nO = 4 * self.nI * wx
        its = np.zeros(R)
        hstride = L_.pt_residuals_stride(C.byref(cfg))  # max_iter + 1 (GMRES) / 2 max_iter + 1 (BiCGstab)
        hist = np.zeros((R, hstride))
        nh = np.zeros(R, dtype=np.int32)
        rel = np.zeros(R)
        conv = np.zeros(R, dtype=np.int32)
        # filled completely by pt_solve (zeros when there is nothing to copy): no zero-fill here
        trac = np.empty((R, max(nO // 2, 1)), dtype=np.complex128)
        pol = np.empty((R, max(nO, 1)), dtype=np.complex128)
        cnt = np.zeros(3, dtype=np.int64)
        ihist = np.zeros(64, dtype=np.int32)
        tms = np.zeros(1)
        kms = np.zeros(3)
        kb = np.zeros(1)
        lc = np.zeros(2, dtype=np.int64)
        cms = np.zeros(5)
        dfl = np.zeros(1)
        cfl = np.zeros(5)
        cby = np.zeros(5)
        st = _abi.PtStats(
            _abi.dptr(its), _abi.dptr(hist), nh.ctypes.data_as(_abi._ip), _abi.dptr(rel),
            conv.ctypes.data_as(_abi._ip), _abi.dptr(trac.view(np.float64)),
            _abi.dptr(pol.view(np.float64)),
            cnt[0:].ctypes.data_as(_abi._llp), cnt[1:].ctypes.data_as(_abi._llp),
            cnt[2:].ctypes.data_as(_abi._llp), ihist.ctypes.data_as(_abi._ip), 64, _abi.dptr(tms),
            _abi.dptr(kms), _abi.dptr(kb), lc[0:].ctypes.data_as(_abi._llp),
            lc[1:].ctypes.data_as(_abi._llp), _abi.dptr(cms), _abi.dptr(dfl), _abi.dptr(cfl), _abi.dptr(cby))
        L = _abi.lib()
        if device_arrays is None:
            F = np.ascontiguousarray(F, dtype=np.complex128)
            if out is not None:
                if out.shape != F.shape or out.dtype != np.complex128 or not out.flags.c_contiguous:
                    raise ValueError("out must be a C-contiguous complex128 array shaped like F")
                U = out
            else:
                U = np.empty_like(F)
            rc = L.pt_solve(self.ctx.handle, _abi.dptr(F.view(np.float64)), R, C.byref(cfg),
                            _abi.dptr(U.view(np.float64)), C.byref(st))
        else:
            fptr, uptr, _ = device_arrays
            U = None
            rc = L.pt_solve_device(self.ctx.handle, C.c_void_p(fptr), R, C.byref(cfg),
                                   C.c_void_p(uptr), C.byref(st))
        self.last_stats = dict(layer_solves=int(cnt[0]), inner_iterations=int(cnt[1]),
                               touches=int(cnt[2]), inner_hist=ihist.copy(), device_ms=float(tms[0]),
                               k1_ms=float(kms[0]), inner_ms=float(kms[1]), other_ms=float(kms[2]),
                               k1_bytes=float(kb[0]), launches=int(lc[0]), k1_launches=int(lc[1]),
                               class_ms=cms.copy(), dense_flops=float(dfl[0]), class_flops=cfl.copy(),
                               class_bytes=cby.copy())
        if rc == _abi.PT_NOT_CONVERGED:
            bad = int(np.argmin(conv))
            h = list(hist[bad, : nh[bad]])
            raise KrylovBreakdown(
                f"trace solve did not reach {config.ktol:g} in {config.max_iter} iterations "
                f"(last residual {h[-1] if h else float('nan'):.3e})", residuals=h)
        if rc != _abi.PT_OK:
            exc = _ERR.get(rc, RuntimeError)
            raise exc(f"pt_solve failed ({rc}): {_abi.last_error()}")
        out = []
        for r in range(R):
            h = [float(v) for v in hist[r, : nh[r]]]
            traces = polar = None
            if self.nI > 0:
                traces = TraceStack(trac[r].reshape(self.nI, 2, wx))
                polar = PolarizedTraceStack.from_flat(pol[r], self.nI, wx)
            u = None if U is None else U[r]
            if self.nI == 0 and not h:
                h = [float(rel[r])]  # monolayer path (sie.py:401-404)
            out.append(SolveResult(u, float(its[r]), h, bool(conv[r]), float(rel[r]),
                                   float(rel[r]) / config.ktol, traces, polar))
        return out

    def solve(self, f_global, config=KrylovConfig(), preconditioner="gs"):
        """``sie.py:392-439``: one source."""
        f = np.asarray(f_global, dtype=complex).reshape(self.grid.shape)
        res = self._run(f[None], config, preconditioner)[0]
        if res.iterations == 0.0 and np.linalg.norm(f) == 0.0:
            res = SolveResult(np.zeros(self.grid.shape, dtype=complex), 0.0, [0.0])
        return res

    def solve_many(self, F, config=KrylovConfig(), preconditioner="gs", out=None):
        """Batch of sources ``F[nrhs, wz, wx]`` solved in lockstep on the device.

        ``out`` (optional, e.g. a pinned buffer) receives the wavefields."""
        F = np.asarray(F, dtype=complex).reshape((-1,) + tuple(self.grid.shape))
        return self._run(F, config, preconditioner, out=out)

    def solve_device(self, f_ptr, u_ptr, nrhs, config=KrylovConfig(), preconditioner="gs"):
        """Device-resident sources/wavefields (e.g. torch CUDA tensors' ``data_ptr()``)."""
        return self._run(None, config, preconditioner, device_arrays=(f_ptr, u_ptr, nrhs))

    # -- test hooks on the same device factors
    def layer_solve(self, layer, rhs, inner_ktol=None, inner_max_iter=None):
        """``NestedLayerSolver.solve`` (nested.py:344-353) for volumes [nrhs, w, wx]."""
        rhs = np.ascontiguousarray(np.asarray(rhs, dtype=np.complex128))
        if rhs.ndim == 2:
            rhs = rhs[None]
        out = np.empty_like(rhs)
        st = _abi.PtStats()
        rc = _abi.lib().pt_layer_solve(
            self.ctx.handle, int(layer), _abi.dptr(rhs.view(np.float64)), rhs.shape[0],
            float(inner_ktol if inner_ktol is not None else self.layers.inner_ktol),
            int(inner_max_iter if inner_max_iter is not None else self.layers.inner_max_iter),
            _abi.dptr(out.view(np.float64)), C.byref(st))
        if rc != _abi.PT_OK:
            raise _ERR.get(rc, RuntimeError)(f"pt_layer_solve failed ({rc}): {_abi.last_error()}")
        return out

    def cell_solve(self, layer, cell, b):
        """One cell's ``LayerWorkspace.solve`` (subdomain.py:214-221) via K1: b [nrhs, wz_c, w]."""
        b = np.ascontiguousarray(np.asarray(b, dtype=np.complex128))
        if b.ndim == 2:
            b = b[None]
        x = np.empty_like(b)
        rc = _abi.lib().pt_cell_solve(self.ctx.handle, int(layer), int(cell),
                                      _abi.dptr(b.view(np.float64)), b.shape[0],
                                      _abi.dptr(x.view(np.float64)))
        if rc != _abi.PT_OK:
            raise RuntimeError(f"pt_cell_solve failed ({rc}): {_abi.last_error()}")
        return x
