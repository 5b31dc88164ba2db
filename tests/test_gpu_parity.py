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


@pytest.mark.parametrize("method,max_iter", [("bicgstab", 2), ("bicgstab", 3), ("gmres", 2)])
def test_unconverged_residual_history_matches_oracle(method, max_iter):
    """A run that stops at max_iter keeps its WHOLE residual history: BiCGstab records the initial 1.0 and
    two half steps per iteration (krylov.py:159-199), i.e. up to 2 max_iter + 1 entries, GMRES up to
    max_iter + 1 (pt_residuals_stride).  The KrylovBreakdown carries the list of the reference's own
    non-converged solve (sie.py:420-425)."""
    from oracle.polartraces_oracle import KrylovBreakdown as OracleBreakdown
    from paper_1510_01831_b200 import KrylovBreakdown

    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3)
    dev = device_solver(prob)
    orc = OracleSolver.from_problem(prob)
    f = prob.rhs([1])[0]
    with pytest.raises(OracleBreakdown) as want:
        orc.solve(f, ktol=1e-15, max_iter=max_iter, method=method)
    with pytest.raises(KrylovBreakdown) as got:
        dev.solve(f, KrylovConfig(ktol=1e-15, max_iter=max_iter, method=method))
    w, g = list(want.value.residuals), list(got.value.residuals)
    assert len(g) == len(w), (g, w)
    if method == "bicgstab":
        assert len(g) == 2 * max_iter + 1
    np.testing.assert_allclose(g, w, rtol=1e-6, atol=1e-15)
    assert f"{w[-1]:.3e}" in str(got.value)


# ---------------------------------------------------------------------------------------------------------------
# Per-source parity of the many-RHS source sets.  tests/golden/<cfg>_s<k>.npz hold the live
# reference's solve of source k of config <cfg> (tests/golden/make_golden.py `sources`): the wavefield (full
# resolution for cfg1 / cfg2 source 0, decimated otherwise), the outer residual history, relres, the Green-block
# touches, the per-layer-solve inner iteration counts and the reassembled traces (SolveResult.traces,
# sie.py:426-427).  The reference solves every source independently (sie.py:392-439) with its own inner GMRES
# per layer solve (nested.py:134-153); the device batches them in lockstep, so both the single-source and the
# batched device solves must reproduce every fixture.

def _source_fixtures():
    out = []
    for fn in sorted(os.listdir(os.path.join(HERE, "golden"))):
        if "_s" in fn and fn.endswith(".npz") and fn.split("_s")[0] in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
            out.append(fn[:-4])
    return out


SOURCE_FIXTURES = _source_fixtures()


def _check_fixture(res, g, st=None, bar=1e-8):
    d = int(g["decim"])
    err = rel(res.u[::d, ::d], g["u"])
    assert err <= bar, err
    assert res.iterations == float(g["iterations"])
    np.testing.assert_allclose(res.residuals, g["residuals"], rtol=1e-4, atol=1e-15)
    assert abs(res.relative_residual - float(g["relres"])) <= 1e-3 * float(g["relres"]) + 1e-13
    td = int(g["trace_decim"])
    terr = rel(res.traces.data[:, :, ::td], g["traces"])
    assert terr <= bar, terr
    if st is not None:
        want = np.bincount(g["inner_iterations"].astype(int), minlength=64)
        assert np.array_equal(st["inner_hist"][: len(want)], want[:64])
        assert st["touches"] == int(g["touches"])
    return err, terr


def _large_solver(name):
    for key in [k for k in _SOLVERS if k[0] in ("cfg3", "cfg4", "cfg5") and k[0] != name]:
        _SOLVERS.pop(key).close()
    return device_solver(make_config(name))


@pytest.mark.parametrize("fixture", SOURCE_FIXTURES)
def test_single_source_matches_reference_fixture(fixture):
    name, k = fixture.split("_s")
    g = np.load(os.path.join(HERE, "golden", f"{fixture}.npz"))
    assert int(g["src_idx"]) == int(k)
    prob = make_config(name)
    dev = _large_solver(name)
    res = dev.solve(prob.rhs([int(k)])[0], KrylovConfig(ktol=float(g["ktol"]), max_iter=200))
    _check_fixture(res, g, dev.last_stats)


@pytest.mark.parametrize("name,idx", [
    ("cfg2", list(range(16))),
    ("cfg3", list(range(64))),
    # crosses the lockstep batch size and mixes far-apart sources
    ("cfg4", list(range(56)) + [63, 127, 255]),
    # the whole 256-source set: one lockstep batch of 256 where the device memory allows (solver.cu batch_rhs)
    ("cfg4", list(range(256))),
    ("cfg5", list(range(64))),
])
def test_batched_sources_match_single_solves_and_fixtures(name, idx):
    """All sources of the set in ONE solve_many call: every fixture source matches the reference, and a sample
    of batched sources equals its own single-source device solve (u to 1e-13, identical outer iterations and
    residual histories) -- lockstep batching with convergence compaction must not couple sources."""
    prob = make_config(name)
    dev = _large_solver(name)
    cfg = KrylovConfig(ktol=prob.ktol, max_iter=200)
    F = prob.rhs(idx)
    many = dev.solve_many(F, cfg)
    assert all(r.converged for r in many)
    fixtures = [f for f in SOURCE_FIXTURES if f.split("_s")[0] == name]
    checked = 0
    for fx in fixtures:
        k = int(fx.split("_s")[1])
        if k in idx:
            _check_fixture(many[idx.index(k)], np.load(os.path.join(HERE, "golden", f"{fx}.npz")))
            checked += 1
    assert checked >= 1
    # iterations within +-1 of the reference for every source with a fixture; sample single solves
    sample = sorted({0, len(idx) // 3, len(idx) - 1} | {idx.index(int(f.split("_s")[1])) for f in fixtures
                                                         if int(f.split("_s")[1]) in idx})
    for r in sample:
        one = dev.solve(F[r], cfg)
        assert rel(many[r].u, one.u) < 1e-13, (r, rel(many[r].u, one.u))
        assert many[r].iterations == one.iterations
        # the last entries sit at the rounding floor (~1e-13 of beta0): compare them absolutely
        np.testing.assert_allclose(many[r].residuals, one.residuals, rtol=1e-6, atol=1e-12)
        assert rel(many[r].traces.data, one.traces.data) < 1e-13


@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_batched_inner_histogram_is_sum_of_single_histograms(name):
    """The inner GMRES of every (layer solve, source) instance stops on its own residual: the batched solve's
    inner iteration histogram and Green-block touches equal the sums over single-source solves."""
    prob = make_config(name)
    dev = _large_solver(name)
    cfg = KrylovConfig(ktol=prob.ktol, max_iter=200)
    idx = [0, 9, 21, 33, 42, 50, 63, 5]
    F = prob.rhs(idx)
    dev.solve_many(F, cfg)
    hist_b, touch_b = dev.last_stats["inner_hist"].copy(), dev.last_stats["touches"]
    hist_s, touch_s = np.zeros_like(hist_b), 0
    for f in F:
        dev.solve(f, cfg)
        hist_s += dev.last_stats["inner_hist"]
        touch_s += dev.last_stats["touches"]
    assert np.array_equal(hist_b, hist_s)
    assert touch_b == touch_s


def test_solve_with_factors_built_from_reference_objects():
    """Drop-in construction (sie.py:368-390): the factors from the reference's own build_nested_layers objects
    (couplings read from their operators, their GreenBlockSet matrices; tests/golden/make_refobj.py) solve like
    the oracle on the device, and global_operator feeds the true residual."""
    from paper_1510_01831_b200.artifacts import load_offline
    from paper_1510_01831_b200.discretization import assemble_fd
    from tests.golden_cases import REFOBJ_CASE

    prob = small_problem(**REFOBJ_CASE)
    layers = load_offline(os.path.join(HERE, "golden", "refobj"), "refobj", prob.grid, prob.partition,
                          model=prob.model, omega=prob.pml.omega)
    H = assemble_fd(prob.grid, prob.model, prob.pml)
    dev = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers, global_operator=H)
    orc = OracleSolver.from_problem(prob)
    for f in prob.rhs():
        got = dev.solve(f, KrylovConfig(ktol=1e-9))
        want = orc.solve(f, ktol=1e-9)
        assert rel(got.u, want.u) < 1e-10
        assert got.iterations == want.iterations
        assert abs(got.relative_residual - want.relative_residual) <= 1e-6 * want.relative_residual + 1e-14
    assert dev.global_operator() is H
    dev.close()


@pytest.mark.parametrize("case", [dict(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), "cfg1", "cfg2"])
def test_offline_operators_by_k1_match_torch_block_substitution(case):
    """the Green blocks (GreenBlockSet.build, green.py:103-129), sampled trace responses and
    pass-0 operators built as many-RHS solves of the repo's own K1 kernel (cell_solver="k1", the default on a
    CUDA device) equal the torch block substitution on the same device to 1e-12, and the reference construction
    on the host."""
    import torch

    from paper_1510_01831_b200.offline import build_factors

    prob = small_problem(**case) if isinstance(case, dict) else make_config(case)
    args = (prob.grid, prob.model, prob.pml, prob.partition, prob.Lc)
    Fk = build_factors(*args, device="cuda", cell_solver="k1")
    Ft = build_factors(*args, device="cuda", cell_solver="torch")
    Fh = build_factors(*args, device="cpu")
    for lk, lt, lh in zip(Fk.layers, Ft.layers, Fh.layers):
        for ck, ct, ch in zip(lk.cells, lt.cells, lh.cells):
            for name in ("green", "gsmp", "q0"):
                a, b, c = getattr(ck, name), getattr(ct, name), getattr(ch, name)
                assert a.shape == b.shape and a.is_cuda
                scale = float(torch.linalg.norm(b))
                assert float(torch.linalg.norm(a - b)) <= 1e-12 * scale, (lk.index, ck.cell, name)
                assert float(torch.linalg.norm(a.cpu() - c)) <= 1e-12 * scale, (lk.index, ck.cell, name)
        if lt.dense is not None:
            assert float(torch.linalg.norm(lk.dense - lt.dense)) <= 1e-11 * float(torch.linalg.norm(lt.dense))


def test_solve_with_plr_compressed_reference_layers():
    """Reference layers built with PLR-compressed Green blocks (plr.py, nested.py:279-307): the factors built from
    those objects (blocks expanded by GreenBlockSet.dense; tests/golden/make_refobj.py) reproduce the reference's
    own solves WITH its compressed layers (it applies U (V x), the device (U V) x)."""
    from paper_1510_01831_b200.artifacts import load_offline
    from tests.golden_cases import REFOBJ_CASE

    prob = small_problem(**REFOBJ_CASE)
    layers = load_offline(os.path.join(HERE, "golden", "refobj_plr"), "refobj_plr", prob.grid, prob.partition,
                          model=prob.model, omega=prob.pml.omega)
    dev = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
    g = np.load(os.path.join(HERE, "golden", "refobj_plr.npz"))
    for k, f in enumerate(prob.rhs()):
        got = dev.solve(f, KrylovConfig(ktol=1e-9))
        assert rel(got.u, g["u"][k]) <= 1e-8
        assert got.iterations == float(g["iterations"][k])
        assert abs(got.relative_residual - float(g["relres"][k])) <= 1e-3 * float(g["relres"][k]) + 1e-13
    dev.close()


def test_source_set_larger_than_the_lockstep_batch():
    """More sources than one lockstep batch holds (pt_solve cuts the set into consecutive batches and moves the
    neighbouring batches' host copies on a side stream while a batch solves): every sampled source -- first and
    last of a batch, and the sources either side of a batch boundary -- equals its own single-source solve and the
    oracle; the counters add up over the batches."""
    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3, n_sources=700)
    dev = device_solver(prob)
    orc = OracleSolver.from_problem(prob)
    cfg = KrylovConfig(ktol=1e-9)
    F = prob.rhs()
    out = np.empty_like(F)
    many = dev.solve_many(F, cfg, out=out)
    assert len(many) == 700 and all(r.converged for r in many)
    assert dev.last_stats["layer_solves"] > 0 and dev.last_stats["inner_hist"].sum() > 0
    # batch sizes of this path: 64 (item programs) or 8 * floor(256 / widest stage) = 336 (dense, L = 4)
    for r in (0, 63, 64, 127, 128, 335, 336, 337, 671, 672, 699):
        one = dev.solve(F[r], cfg)
        assert rel(many[r].u, one.u) < 1e-13, r
        assert many[r].u is not None and np.array_equal(many[r].u, out[r])
        assert many[r].iterations == one.iterations
        np.testing.assert_allclose(many[r].residuals, one.residuals, rtol=1e-6, atol=1e-12)
    for r in (0, 336, 699):
        want = orc.solve(F[r], ktol=1e-9)
        assert rel(many[r].u, want.u) < 1e-10
        assert many[r].iterations == want.iterations
