"""GPU parity: the B200 path (through the C ABI) against the oracle and the
live-reference golden fixtures.

Bars (BASELINE.json north_star): wavefield relative L2 error <= 1e-8 in
complex128, outer GMRES iterations within +-1 (we require equality where the
reference's residual margin allows), inner per-layer-solve iteration counts
identical as a multiset (the inner Krylov process must be replicated,
SURVEY.md 8(c)).  Cell solves vs SuperLU: 1e-12; layer solves vs the oracle's
NestedLayerSolver: 1e-10.
"""

import os

import numpy as np
import pytest

from oracle.polartraces_oracle import OracleSolver
from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers
from paper_1510_01831_b200.configs import make_config, small_problem
from tests.golden_cases import GOLDEN

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
_SOLVERS = {}


def device_solver(prob, nested=True, backend="pt", assembled=False):
    key = (prob.name, prob.Lc if nested else 1, id(prob) if prob.name.startswith("tmp") else 0, backend, assembled)
    if key not in _SOLVERS:
        Lc = prob.Lc if nested else 1
        # the large configs run their offline arithmetic on the GPU (torch), the small ones on the host
        dev = "cuda" if prob.name in ("cfg3", "cfg4", "cfg5") else "cpu"
        layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=Lc,
                                     inner_ktol=prob.inner_ktol, device=dev, backend=backend,
                                     assembled_boundary=assembled)
        _SOLVERS[key] = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition,
                                              layers=layers)
    return _SOLVERS[key]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_k1_cell_solve_matches_superlu():
    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3)
    dev = device_solver(prob)
    orc = OracleSolver.from_problem(prob)
    rng = np.random.default_rng(0)
    for l, lay in enumerate(orc.outer.slabs):
        for c, cell in enumerate(lay.cells):
            b = rng.standard_normal((11,) + cell.shape) + 1j * rng.standard_normal((11,) + cell.shape)
            x = dev.cell_solve(l, c, b)
            for r in range(b.shape[0]):
                assert rel(x[r], cell.solve(b[r])) < 1e-12


@pytest.mark.parametrize("case", [dict(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3),
                                  dict(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7),
                                  dict(nx=40, nz=36, npml=6, L=3, Lc=1, omega=14.0, seed=0)])
def test_layer_solve_matches_nested_layer_solver(case):
    """NestedLayerSolver.solve (nested.py:344-353): swap, cells, inner PT GMRES, rebuild."""
    prob = small_problem(**case)
    dev = device_solver(prob)
    orc = OracleSolver.from_problem(prob)
    rng = np.random.default_rng(5)
    for l, lay in enumerate(orc.outer.slabs):
        f = rng.standard_normal((3,) + lay.shape) + 1j * rng.standard_normal((3,) + lay.shape)
        f[2] = 0.0
        f[2, lay.row(1), 4] = 1.0 / prob.grid.h**2
        out = dev.layer_solve(l, f)
        for r in range(3):
            want = lay.solve(f[r]) if hasattr(lay, "cells") else lay.solve(f[r])
            assert rel(out[r], want) < 1e-10, (l, r, rel(out[r], want))


@pytest.mark.parametrize("name", ["small_a", "small_b", "small_c", "small_direct", "cfg1", "cfg2", "cfg3",
                                  "cfg4", "cfg5", "small_b_bicgstab", "cfg1_bicgstab", "small_b_lu", "small_c_lu",
                                  "cfg1_lu", "cfg2_lu", "small_b_asm", "small_c_asm", "cfg1_asm"])
def test_solve_matches_reference_fixture(name):
    make, si, nested = GOLDEN[name]
    prob = make()
    for key in [k for k in _SOLVERS if k[0] in ("cfg3", "cfg4", "cfg5") and k[0] != name]:
        _SOLVERS.pop(key).close()  # the large configs hold tens of GB of factors each
    g = np.load(os.path.join(HERE, "golden", f"{name}.npz"))
    dev = device_solver(prob, nested, str(g["backend"]) if "backend" in g.files else "pt",
                        bool(g["assembled"]) if "assembled" in g.files else False)
    method = str(g["method"]) if "method" in g.files else "gmres"
    res = dev.solve(prob.rhs([si])[0], KrylovConfig(ktol=float(g["ktol"]), max_iter=200, method=method))
    d = int(g["decim"])
    err = rel(res.u[::d, ::d], g["u"])
    assert err <= 1e-8, err
    assert res.iterations == float(g["iterations"])
    np.testing.assert_allclose(res.residuals, g["residuals"], rtol=1e-4, atol=1e-15)
    assert abs(res.relative_residual - float(g["relres"])) <= 1e-3 * float(g["relres"]) + 1e-13
    assert abs(np.linalg.norm(res.u) - float(g["unorm"])) <= 1e-9 * float(g["unorm"])
    if nested:
        st = dev.last_stats
        want = np.bincount(g["inner_iterations"].astype(int), minlength=64)
        got = st["inner_hist"][: len(want)]
        assert np.array_equal(got, want[: len(got)]), (got[:8], want[:8])
        assert st["touches"] == int(g["touches"])


def test_solve_many_matches_single_solves_and_oracle():
    prob = make_config("cfg2")
    dev = device_solver(prob)
    F = prob.rhs([0, 5, 11])
    many = dev.solve_many(F, KrylovConfig(ktol=1e-9))
    for r, idx in enumerate([0, 5, 11]):
        one = dev.solve(F[r], KrylovConfig(ktol=1e-9))
        assert rel(many[r].u, one.u) < 1e-13
        assert many[r].iterations == one.iterations
    g = np.load(os.path.join(HERE, "golden", "cfg2.npz"))
    assert rel(many[0].u[::8, ::8], g["u"]) <= 1e-8


def test_zero_source_and_mixed_batch():
    prob = small_problem(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0, seed=0)
    dev = device_solver(prob)
    res = dev.solve(np.zeros(prob.grid.shape), KrylovConfig(ktol=1e-9))
    assert res.iterations == 0.0 and np.linalg.norm(res.u) == 0.0 and res.residuals == [0.0]
    F = prob.rhs([0, 1])
    F[1] = 0.0
    out = dev.solve_many(F, KrylovConfig(ktol=1e-9))
    assert np.linalg.norm(out[1].u) == 0.0
    orc = OracleSolver.from_problem(prob)
    assert rel(out[0].u, orc.solve(F[0], ktol=1e-9).u) < 1e-10


@pytest.mark.parametrize("precond,restart", [("jac", 0), ("gs", 2)])
def test_jacobi_and_restarted_gmres_match_oracle(precond, restart):
    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3)
    dev = device_solver(prob)
    orc = OracleSolver.from_problem(prob)
    f = prob.rhs([1])[0]
    want = orc.solve(f, ktol=1e-9, restart=restart, preconditioner=precond)
    got = dev.solve(f, KrylovConfig(ktol=1e-9, restart=restart), preconditioner=precond)
    assert got.iterations == want.iterations
    assert rel(got.u, want.u) < 1e-9
    np.testing.assert_allclose(got.residuals, want.residuals, rtol=1e-5, atol=1e-15)


def test_monolayer_and_one_cell():
    prob = small_problem(nx=30, nz=14, npml=4, L=1, Lc=2, omega=9.0, seed=4)
    dev = device_solver(prob)
    orc = OracleSolver.from_problem(prob)
    f = prob.rhs([0])[0]
    got = dev.solve(f, KrylovConfig(ktol=1e-9))
    want = orc.solve(f, ktol=1e-9)
    assert got.iterations == 0.0
    assert rel(got.u, want.u) < 1e-10


@pytest.mark.parametrize("name", ["small_b", "cfg1", "cfg2"])
def test_repeated_solves_replay_graphs(name):
    """The fixed launch sequences of a solve run eagerly the first time, are captured as CUDA graphs the
    second time and replayed after that: all three must give the same wavefield (bitwise: same kernels,
    same order) and the same counters, matching the live-reference fixture."""
    make, si, nested = GOLDEN[name]
    prob = make()
    g = np.load(os.path.join(HERE, "golden", f"{name}.npz"))
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc,
                                 inner_ktol=prob.inner_ktol)
    dev = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
    f = prob.rhs([si])[0]
    cfg = KrylovConfig(ktol=float(g["ktol"]), max_iter=200)
    outs, stats = [], []
    for _ in range(4):
        r = dev.solve(f, cfg)
        outs.append(r.u.copy())
        stats.append((r.iterations, dev.last_stats["touches"], dev.last_stats["layer_solves"],
                      dev.last_stats["launches"]))
    for k in range(1, 4):
        assert np.array_equal(outs[k], outs[0])
        assert stats[k] == stats[0], (stats[k], stats[0])
    d = int(g["decim"])
    assert rel(outs[-1][::d, ::d], g["u"]) <= 1e-8
    dev.close()
