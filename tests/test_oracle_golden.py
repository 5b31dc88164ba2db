"""CPU: the oracle (oracle/polartraces_oracle.py) against the live-reference fixtures.

The fixtures were produced by tests/golden/make_golden.py running the
reference itself; the oracle must reproduce them bit for bit (same arithmetic,
same SuperLU), and the config-1/2 anchors of SURVEY.md section 8(c).
"""

import os

import numpy as np
import pytest

from oracle.polartraces_oracle import OracleSolver
from tests.golden_cases import GOLDEN

HERE = os.path.dirname(os.path.abspath(__file__))


def load(name):
    return np.load(os.path.join(HERE, "golden", f"{name}.npz"))


@pytest.mark.parametrize("name", ["small_a", "small_b", "small_c", "small_direct", "cfg1", "small_b_bicgstab",
                                  "cfg1_bicgstab", "small_b_lu", "small_c_lu", "cfg1_lu"])
def test_oracle_matches_reference_fixture(name):
    make, si, nested = GOLDEN[name]
    prob = make()
    g = load(name)
    backend = str(g["backend"]) if "backend" in g.files else "pt"
    s = OracleSolver.from_problem(prob, nested=nested, backend=backend)
    method = str(g["method"]) if "method" in g.files else "gmres"
    r = s.solve(prob.rhs([si])[0], ktol=float(g["ktol"]), method=method)
    d = int(g["decim"])
    u = r.u[::d, ::d]
    assert np.array_equal(u, g["u"]), np.abs(u - g["u"]).max()
    assert r.iterations == float(g["iterations"])
    assert np.array_equal(np.array(r.residuals), g["residuals"])
    assert r.relative_residual == float(g["relres"])
    assert r.touches == int(g["touches"])
    inner = sorted(x for lay in r.inner_iterations for x in lay)
    assert inner == sorted(g["inner_iterations"].tolist())


def test_cfg1_known_answer_anchors():
    """2 iterations, residuals [3.110e-07, 2.076e-13], relres 8.786e-09,
    ||u|| = 6.266714, u[row(120), col(80)], touches 3,830,400."""
    g = load("cfg1")
    assert float(g["iterations"]) == 2.0
    np.testing.assert_allclose(g["residuals"], [3.110e-07, 2.076e-13], rtol=2e-3)
    assert abs(float(g["relres"]) - 8.786e-09) < 1e-12
    assert abs(float(g["unorm"]) - 6.266714) < 1e-6
    assert int(g["touches"]) == 3_830_400
    grid_row, grid_col = 120 + 10 - 1, 80 + 10 - 1
    v = g["u"][grid_row // 4, grid_col // 4] if grid_row % 4 == 0 and grid_col % 4 == 0 else None
    if v is not None:
        assert abs(v - (0.0072115656 + 0.0280498056j)) < 1e-9


def test_cfg2_known_answer_anchors():
    g = load("cfg2")
    assert float(g["iterations"]) == 3.0
    np.testing.assert_allclose(g["residuals"], [2.132e-04, 3.578e-09, 1.279e-13], rtol=2e-3)
    assert abs(float(g["relres"]) - 3.814e-10) < 1e-13
    assert abs(float(g["unorm"]) - 10.37541) < 1e-5
    assert int(g["touches"]) == 118_227_200
    assert len(g["inner_iterations"]) == 134  # N_ls = 2L + (3L-5) + k(5L-7), L=8, k=3


@pytest.mark.parametrize("name,L,its", [("cfg3", 16, 7), ("cfg4", 20, 9), ("cfg5", 32, 11)])
def test_large_config_fixtures_are_consistent(name, L, its):
    """cfg3-5 fixtures (live reference, one source each; too slow to re-run the oracle here): the outer
    iteration count, a monotone residual history ending below ktol, and one inner GMRES per layer solve,
    N_ls = 2L + (3L-5) + k(5L-7)."""
    g = load(name)
    k = int(g["iterations"])
    assert k == its
    r = np.asarray(g["residuals"])
    assert len(r) == k and r[-1] <= float(g["ktol"]) and np.all(np.diff(r) < 0)
    assert len(g["inner_iterations"]) == 2 * L + (3 * L - 5) + k * (5 * L - 7)
    assert float(g["relres"]) < 1e-5
