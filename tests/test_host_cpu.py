"""CPU: host-side logic -- value types, partitions, config generators, offline factors,
the C-ABI library exports.  No compute call into the library here (no GPU)."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

from oracle.polartraces_oracle import OracleSolver
from paper_1510_01831_b200 import (
    Grid,
    KrylovConfig,
    PmlProfile,
    VelocityModel,
    default_pml_strength,
    delta_source,
    partition_cells,
    partition_layers,
)
from paper_1510_01831_b200.configs import make_config, small_problem
from paper_1510_01831_b200.offline import _twisted_solve, build_factors

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_partitions_match_reference_rule():
    # subdomain.py:88-110: near-equal, remainder first
    assert partition_layers(Grid(10, 41, 0.1, 2), 4).extents == (11, 10, 10, 10)
    assert partition_layers(Grid(10, 41, 0.1, 2), 4).offsets == (0, 11, 21, 31)
    assert partition_cells(Grid(33, 10, 0.1, 2), 4).extents == (9, 8, 8, 8)
    with pytest.raises(ValueError):
        partition_layers(Grid(10, 5, 0.1, 2), 3)
    with pytest.raises(ValueError):
        partition_cells(Grid(5, 10, 0.1, 2), 3)


def test_value_types_validate_like_reference():
    with pytest.raises(ValueError):
        Grid(0, 5, 0.1, 2)
    with pytest.raises(ValueError):
        PmlProfile(4, 0.1, -1.0, 3.0)
    g = Grid(8, 6, 0.1, 2)
    with pytest.raises(ValueError):
        VelocityModel(g, np.ones((3, 3)))
    with pytest.raises(ValueError):
        KrylovConfig(ktol=0.0)
    with pytest.raises(ValueError):
        delta_source(g, (100, 1))
    f = delta_source(g, (3, 2))
    assert f[g.row_of(2), g.col_of(3)] == 1.0 / 0.1**2


def test_config_generators_are_deterministic_and_match_survey_conventions():
    p1 = make_config("cfg1")
    assert p1.sources == [(80, 40)]
    assert abs(p1.pml.C - 20.723266) < 1e-6
    assert p1.partition.extents == (40, 40, 40, 40)
    p2 = make_config("cfg2")
    assert p2.sources[0] == (244, 40)
    assert abs(p2.pml.omega - 188.966798) < 1e-5
    assert len(p2.sources) == 16
    p2b = make_config("cfg2")
    assert p2b.sources == p2.sources and np.array_equal(p2b.model.c, p2.model.c)


@pytest.mark.parametrize("case", [dict(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3),
                                  dict(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7)])
def test_offline_factors_reproduce_superlu_cells_and_green_blocks(case):
    """Twisted Schur factors solve every cell like SuperLU (1e-12), Green blocks equal the
    reference's GreenBlockSet construction (green.py:103-129) to 1e-12."""
    prob = small_problem(**case)
    F = build_factors(prob.grid, prob.model, prob.pml, prob.partition, prob.Lc)
    O = OracleSolver.from_problem(prob)
    rng = np.random.default_rng(1)
    slots = ("v0", "v1", "vn", "vnp")
    for lf, ol in zip(F.layers, O.outer.slabs):
        for cf, oc in zip(lf.cells, ol.cells):
            n = oc.n
            for jr, j in enumerate((0, 1, n, n + 1)):
                for s, sl in enumerate(slots):
                    A = oc.G[(j, sl)]
                    B = cf.green[jr, s].numpy().T
                    assert np.abs(A - B).max() <= 1e-12 * np.abs(A).max()
            b = rng.standard_normal((cf.wzc, cf.w)) + 1j * rng.standard_normal((cf.wzc, cf.w))
            x0 = oc.solve(b)
            sinv = cf.sinv.transpose(-1, -2)[None]
            x1 = _twisted_solve(sinv, cf.lz, cf.uz, torch.tensor(b)[None, :, :, None])[0, :, :, 0].numpy()
            assert np.linalg.norm(x1 - x0) <= 1e-12 * np.linalg.norm(x0)


def test_cut_coupling_blocks_are_minus_identity_over_h2():
    """all four cut coupling blocks are -I/h^2 for layers and cells."""
    prob = small_problem(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0)
    F = build_factors(prob.grid, prob.model, prob.pml, prob.partition, prob.Lc, green=False)
    h2 = prob.grid.h ** 2
    for lf in F.layers:
        np.testing.assert_allclose(lf.coefs * h2, [1, -1, -1, 1], atol=1e-14)
        for cf in lf.cells:
            np.testing.assert_allclose(cf.coefs * h2, [1, -1, -1, 1], atol=1e-14)


def _header_symbols():
    txt = open(os.path.join(REPO, "include", "pt_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(pt_\w+)\(", txt, re.M)))


def test_c_abi_library_exports_every_header_symbol():
    from paper_1510_01831_b200 import _abi
    from paper_1510_01831_b200.build import build

    build()
    lib = ctypes.CDLL(_abi.LIB_PATH)
    syms = _header_symbols()
    assert set(syms) == set(_abi.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert b"sm_100a" in _abi.lib().pt_version()


def test_ctypes_structs_match_the_c_header(tmp_path):
    """The ctypes mirrors of pt_problem / pt_krylov / pt_stats have the header's size and field offsets
    (a C program compiled against include/pt_b200.h prints them)."""
    import subprocess

    from paper_1510_01831_b200 import _abi

    structs = {"pt_problem": _abi.PtProblem, "pt_krylov": _abi.PtKrylov, "pt_stats": _abi.PtStats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pt_b200.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True,
                                                   check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_solver_fails_loudly_without_gpu():
    """No CPU fallback: constructing the device solver without a GPU raises."""
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1510_01831_b200 import PolarizedTracesSolver, build_nested_layers

    prob = small_problem(nx=20, nz=16, npml=4, L=2, Lc=2)
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=2)
    with pytest.raises(RuntimeError):
        PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)


# --- offline operators of the one-pass layer solve and the dense inner GMRES (CPU, torch) -----------

def _offline_case():
    from paper_1510_01831_b200.configs import small_problem
    from paper_1510_01831_b200.offline import build_factors

    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3)
    return prob, build_factors(prob.grid, prob.model, prob.pml, prob.partition, 3)


def _cell_solve(cf, rhs):
    import torch

    from paper_1510_01831_b200.offline import _twisted_solve

    tinv = cf.sinv.transpose(-1, -2)  # stored column-major blocks -> row-major twisted factors
    x = _twisted_solve(tinv[None], cf.lz, cf.uz, torch.as_tensor(rhs)[None, :, :, None])
    return x[0, :, :, 0].numpy()


def test_pass0_operator_matches_cell_solves():
    """Q0 (offline.py) = the first layer-solve pass without volume source: Newton rows + trace samples."""
    prob, F = _offline_case()
    npml = F.npml
    rng = np.random.default_rng(0)
    for lf in F.layers:
        for ci, cf in enumerate(lf.cells):
            lo = 0 if ci == 0 else npml
            hi = cf.wzc if ci == len(lf.cells) - 1 else npml + cf.nxc
            nk, nk4 = hi - lo, (hi - lo + 3) // 4 * 4
            P = rng.standard_normal((4, nk)) + 1j * rng.standard_normal((4, nk))
            rhs = np.zeros((cf.wzc, cf.w), complex)
            for s in range(4):
                rhs[lo:hi, lf.prows[s]] += lf.coefs[s] * P[s]
            x = _cell_solve(cf, rhs)
            rows4 = [int(r) for r in (cf.krows[1], cf.krows[0], cf.krows[3], cf.krows[2])]
            jrows = [npml - 1, npml, lf.n + npml - 1, lf.n + npml]
            want = np.concatenate([x[rows4].reshape(-1), x[lo:hi][:, jrows].reshape(-1)])
            Pp = np.zeros((4, nk4), complex)
            Pp[:, :nk] = P
            got = cf.q0.numpy()[: 4 * cf.w + 4 * nk] @ Pp.reshape(-1)
            assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_sampled_trace_response_matches_cell_solves():
    """gsmp (offline.py): the trace-source response sampled at the layer trace rows, every block row."""
    prob, F = _offline_case()
    npml = F.npml
    rng = np.random.default_rng(1)
    for lf in F.layers:
        for cf in lf.cells:
            tr = rng.standard_normal((4, cf.w)) + 1j * rng.standard_normal((4, cf.w))
            rhs = np.zeros((cf.wzc, cf.w), complex)
            for s in range(4):
                rhs[int(cf.krows[s])] += cf.coefs[s] * tr[s]
            x = _cell_solve(cf, rhs)
            jrows = [npml - 1, npml, lf.n + npml - 1, lf.n + npml]
            want = x[:, jrows]  # (wzc, 4)
            got = np.einsum("kosj,sj->ko", cf.gsmp.numpy(), tr)
            assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_dense_inner_operators_match_oracle():
    """pre and pre o op of the inner trace problem (sie.py:203-329) as dense matrices."""
    from oracle.polartraces_oracle import OracleSolver

    prob, F = _offline_case()
    orc = OracleSolver.from_problem(prob)
    rng = np.random.default_rng(2)
    for l, lf in enumerate(F.layers):
        op, pre, _ = orc.outer.slabs[l].inner.flat_ops("gs")
        Pm, Bm, S1, S2 = (m.numpy() for m in lf.dense)
        v = rng.standard_normal(Pm.shape[0]) + 1j * rng.standard_normal(Pm.shape[0])
        for got, want in ((Pm @ v, pre(v)), (Bm @ v, pre(op(v)))):
            assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
        # s-step operators: E pre and E^2 pre with E = pre o op - I
        b = pre(v)
        e1 = pre(op(b)) - b
        e2 = pre(op(e1)) - e1
        assert np.abs(S1 @ v - e1).max() <= 1e-11 * np.abs(b).max()
        assert np.abs(S2 @ v - e2).max() <= 1e-11 * np.abs(b).max()


def test_inner_lu_inverse_matches_block_lu():
    """backend="lu": the offline inverse of the assembled cell-interface system applies the same linear map
    as the reference's block-LU substitutions (nested.py:156-254, restated in the oracle's InnerLU)."""
    import torch

    from oracle.polartraces_oracle import OracleSolver
    from paper_1510_01831_b200.configs import small_problem
    from paper_1510_01831_b200.offline import build_factors

    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3)
    F = build_factors(prob.grid, prob.model, prob.pml, prob.partition, prob.Lc, backend="lu")
    orc = OracleSolver.from_problem(prob, backend="lu")
    rng = np.random.default_rng(2)
    for ell, lay in enumerate(orc.outer.slabs):
        Ainv = F.layers[ell].lu_inv.numpy()
        w = lay.lu.w
        b = [rng.standard_normal(2 * w) + 1j * rng.standard_normal(2 * w) for _ in range(lay.lu.nI)]
        x = np.concatenate(lay.lu.solve(b))
        y = Ainv @ np.concatenate(b)
        assert np.linalg.norm(y - x) <= 1e-11 * np.linalg.norm(x)
        assert F.layers[ell].dense is None


# ---------------------------------------------------------------------------------------------------------------
# Drop-in construction from the reference's own offline objects (sie.py:368-390, nested.py:272-319, 507-521).
# Skipped where the reference package is absent (the GPU box).

REF_SRC = "/root/reference/pkg/src"


def _reference_objects(prob, Lc=None, backend="pt"):
    import sys

    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import polartraces as rpt

    g = prob.grid
    grid = rpt.Grid(g.nx, g.nz, g.h, g.npml)
    model = rpt.VelocityModel(grid, prob.model.c)
    pml = rpt.PmlProfile(g.npml, g.h, prob.pml.C, prob.pml.omega)
    part = rpt.LayerPartition(tuple(prob.partition.extents))
    if Lc is None:  # direct LayerWorkspace layers (the reference's layers=None default)
        layers = [rpt.build_layer(grid, model, pml, part, ell) for ell in range(1, part.L + 1)]
    else:
        layers = rpt.build_nested_layers(grid, model, pml, part, Lc=Lc, backend=backend,
                                         inner_ktol=prob.inner_ktol)
    return rpt, layers, rpt.discretization.assemble_fd(grid, model, pml)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
@pytest.mark.parametrize("case,Lc,backend", [
    (dict(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 3, "pt"),
    (dict(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7), 4, "lu"),
    (dict(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0, seed=0), None, "pt"),
])
def test_factors_from_reference_objects_equal_own_offline(case, Lc, backend):
    """The arrays uploaded for the reference's own layer objects (couplings read from their assembled
    operators, Green blocks = their GreenBlockSet matrices) equal this package's offline stage to 1e-12."""
    from paper_1510_01831_b200.solver import build_nested_layers, from_reference_layers, is_reference_layers

    prob = small_problem(**case)
    _, ref_layers, _ = _reference_objects(prob, Lc, backend)
    assert is_reference_layers(ref_layers)
    got = from_reference_layers(ref_layers, prob.grid, prob.model, prob.pml, prob.partition)
    want = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=Lc or 1, backend=backend,
                               inner_ktol=prob.inner_ktol)
    assert got.backend == want.backend and got.Lc == want.Lc and got.inner_ktol == want.inner_ktol

    def close(a, b):
        a, b = np.asarray(a), np.asarray(b)
        return np.linalg.norm(a - b) <= 1e-12 * max(np.linalg.norm(b), 1e-300)

    for la, lb in zip(got.factors.layers, want.factors.layers):
        assert close(la.coefs, lb.coefs) and np.array_equal(la.prows, lb.prows)
        for ca, cb in zip(la.cells, lb.cells):
            assert close(ca.lz, cb.lz) and close(ca.uz, cb.uz) and close(ca.coefs, cb.coefs)
            assert np.array_equal(ca.krows, cb.krows)
            assert close(ca.sinv.numpy(), cb.sinv.numpy())
            for name in ("green", "gsmp", "q0"):
                va, vb = getattr(ca, name), getattr(cb, name)
                assert (va is None) == (vb is None)
                if va is not None:
                    assert close(va.numpy(), vb.numpy()), name
        for name in ("dense", "lu_inv"):
            va, vb = getattr(la, name), getattr(lb, name)
            assert (va is None) == (vb is None)
            if va is not None:
                assert close(va.numpy(), vb.numpy()), name


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_global_operator_residual_arrays():
    """global_operator (sie.py:381): the device residual's couplings and diagonal reproduce the caller's H."""
    import scipy.sparse as sp

    from paper_1510_01831_b200.discretization import assemble_fd
    from paper_1510_01831_b200.offline import residual_from_operator

    prob = small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3)
    _, _, Href = _reference_objects(prob, 3)
    H = assemble_fd(prob.grid, prob.model, prob.pml)
    assert abs(H - Href).max() == 0.0  # the restated assembly is the reference's, bit for bit
    g = prob.grid
    tx, tz, hd = residual_from_operator(Href, g.wz, g.wx)
    rebuilt = (sp.kron(sp.eye(g.wz), sp.diags([tx[0][1:], tx[2][:-1]], [-1, 1]))
               + sp.kron(sp.diags([tz[0][1:], tz[2][:-1]], [-1, 1]), sp.eye(g.wx)) + sp.diags(hd.ravel()))
    assert abs(rebuilt - Href).max() == 0.0
    with pytest.raises(ValueError):
        residual_from_operator(Href + sp.eye(Href.shape[0], k=2 * g.wx), g.wz, g.wx)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_plr_compressed_reference_layers_are_accepted():
    """Reference layers built with PLR compression (NestedLayerSolver(plr_threshold=...), nested.py:279-307;
    plr.py:96-219): the uploaded Green blocks are the expansions GreenBlockSet.dense() returns (what the
    reference's own artifact dump stores, green.py:156-163), within the PLR tolerance of the uncompressed ones."""
    import sys

    from paper_1510_01831_b200.solver import build_nested_layers, from_reference_layers
    from tests.golden_cases import REFOBJ_CASE, REFOBJ_PLR

    prob = small_problem(**REFOBJ_CASE)
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import polartraces as rpt

    g = prob.grid
    grid = rpt.Grid(g.nx, g.nz, g.h, g.npml)
    model = rpt.VelocityModel(grid, prob.model.c)
    pml = rpt.PmlProfile(g.npml, g.h, prob.pml.C, prob.pml.omega)
    part = rpt.LayerPartition(tuple(prob.partition.extents))
    ref_layers = rpt.build_nested_layers(grid, model, pml, part, Lc=prob.Lc, inner_ktol=prob.inner_ktol, **REFOBJ_PLR)
    assert any(isinstance(m, rpt.plr.PlrMatrix) for lay in ref_layers for bs in lay.blocksets
               for m in bs.blocks.values())
    got = from_reference_layers(ref_layers, prob.grid, prob.model, prob.pml, prob.partition)
    own = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc, inner_ktol=prob.inner_ktol)
    for lay, la, lo in zip(ref_layers, got.factors.layers, own.factors.layers):
        for bs, ca, co in zip(lay.blocksets, la.cells, lo.cells):
            for jr, jrow in enumerate((0, 1, ca.nxc, ca.nxc + 1)):
                for s, slot in enumerate(("v0", "v1", "vn", "vnp")):
                    dense = np.asarray(bs.dense(jrow, slot))
                    assert np.array_equal(ca.green[jr, s].numpy().T, dense)  # column-major storage
            scale = np.linalg.norm(co.green.numpy())
            err = np.linalg.norm(ca.green.numpy() - co.green.numpy())
            assert err <= 1e-8 * scale  # the compression tolerance (plr_eps = 1e-10 per block, certified)
