"""Krylov configuration/result types of the reference (``krylov.py:17-46``).

The iteration itself runs on the device (outer Arnoldi in ``outer_kernels.cu``
driven by ``solver.cu``; inner GMRES in ``inner_gmres.cu``); only the value
types and exceptions live here so that user code written against the
reference keeps working.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["KrylovConfig", "KrylovResult", "KrylovBreakdown", "InnerSolveError"]


@dataclass(frozen=True)
class KrylovConfig:
    """``krylov.py:17-31``."""

    method: str = "gmres"
    ktol: float = 1e-7
    max_iter: int = 200
    restart: int = 0
    seed: int = 0

    def __post_init__(self):
        if self.ktol <= 0:
            raise ValueError("ktol must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        if self.method not in ("gmres", "bicgstab"):
            raise ValueError(f"unknown Krylov method {self.method!r}")


@dataclass
class KrylovResult:
    x: np.ndarray
    iterations: float
    residuals: list = field(default_factory=list)
    converged: bool = True


class KrylovBreakdown(RuntimeError):
    """``krylov.py:42-46``."""

    def __init__(self, message, basis_size=None, residuals=None):
        super().__init__(message)
        self.basis_size = basis_size
        self.residuals = residuals or []


class InnerSolveError(RuntimeError):
    """``nested.py:50-51``: inner trace solve did not converge."""
