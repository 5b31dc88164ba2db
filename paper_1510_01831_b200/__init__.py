"""B200-native online stage of the nested polarized-traces Helmholtz solver.

Drop-in for the reference's construction + ``solve()`` path
(``/root/reference/pkg/src/polartraces``: ``build_nested_layers`` and
``PolarizedTracesSolver.solve``).  Host code is Python; the online stage runs
in hand-written sm_100a CUDA kernels behind the C ABI in ``include/pt_b200.h``.
"""

from .discretization import (
    CellPartition,
    DiscretizationSpec,
    Grid,
    LayerPartition,
    PmlProfile,
    VelocityModel,
    default_npml,
    default_pml_strength,
    delta_source,
    partition_cells,
    partition_layers,
)
from .krylov import InnerSolveError, KrylovBreakdown, KrylovConfig, KrylovResult
from .artifacts import cache_key, dump_offline, load_model, load_offline, save_model

__version__ = "0.1.0"


def __getattr__(name):
    # the solver imports the C-ABI library lazily so the value types stay importable anywhere
    if name in ("PolarizedTracesSolver", "SolveResult", "TraceStack", "PolarizedTraceStack",
                "build_nested_layers", "NestedLayers"):
        from . import solver

        return getattr(solver, name)
    raise AttributeError(name)


__all__ = [
    "save_model",
    "load_model",
    "cache_key",
    "dump_offline",
    "load_offline",
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
    "KrylovConfig",
    "KrylovResult",
    "KrylovBreakdown",
    "InnerSolveError",
    "PolarizedTracesSolver",
    "SolveResult",
    "TraceStack",
    "PolarizedTraceStack",
    "build_nested_layers",
    "NestedLayers",
]
