"""Formats around the online path: model files and offline artifacts."""

import json

import numpy as np
import pytest
import torch

from oracle.polartraces_oracle import OracleSolver
from paper_1510_01831_b200.artifacts import cache_key, dump_offline, load_model, load_offline, save_model
from paper_1510_01831_b200.configs import small_problem


def _prob():
    return small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3)


def test_model_roundtrip_json_and_csv(tmp_path):
    prob = _prob()
    save_model(tmp_path / "m.json", prob.grid, prob.model)
    hdr = json.loads((tmp_path / "m.json").read_text())
    assert hdr["dtype"] == "f64" and hdr["data"] == "m.bin"
    g, m = load_model(tmp_path / "m.json")
    assert (g.nx, g.nz, g.npml, g.h) == (prob.grid.nx, prob.grid.nz, prob.grid.npml, prob.grid.h)
    assert np.array_equal(m.c, prob.model.c)
    # headered CSV (discretization.py:542-560) on a tiny grid
    from paper_1510_01831_b200.discretization import Grid

    tiny = Grid(3, 2, 0.25, 1)
    c = 1.0 + np.arange(tiny.wz * tiny.wx, dtype=float).reshape(tiny.shape) / 10
    lines = ["# nx=3 nz=2 npml=1 h=0.25"] + [",".join(f"{v:.17g}" for v in row) for row in c]
    (tmp_path / "t.csv").write_text("\n".join(lines))
    g2, m2 = load_model(tmp_path / "t.csv")
    assert g2.shape == tiny.shape and np.array_equal(m2.c, c)
    (tmp_path / "bad.csv").write_text("1,2\n3,4\n")
    with pytest.raises(ValueError):
        load_model(tmp_path / "bad.csv")


def test_cache_key_is_stable_and_sensitive():
    prob = _prob()
    k1 = cache_key(prob.model, prob.grid, prob.pml.omega, prob.partition)
    assert k1 == cache_key(prob.model, prob.grid, prob.pml.omega, prob.partition) and len(k1) == 16
    assert k1 != cache_key(prob.model, prob.grid, prob.pml.omega * 1.01, prob.partition)


def test_dump_offline_reference_format_and_reload(tmp_path):
    from paper_1510_01831_b200 import build_nested_layers

    prob = _prob()
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc)
    key = cache_key(prob.model, prob.grid, prob.pml.omega, prob.partition)
    dump_offline(layers, tmp_path, key, model=prob.model, grid=prob.grid, omega=prob.pml.omega,
                 partition=prob.partition)
    # the Green blocks in GreenBlockSet.dump's format equal the oracle's blocks (green.py:103-129)
    orc = OracleSolver.from_problem(prob)
    for ell, lay in enumerate(orc.outer.slabs):
        for c, cell in enumerate(lay.cells):
            tag = f"{key}_layer{ell + 1}_cell{c + 1}"
            man = json.loads((tmp_path / f"green_{tag}.json").read_text())
            assert man["n"] == cell.n and man["width"] == cell.width
            data = np.load(tmp_path / f"green_{tag}.npz")
            assert len(data.files) == 16
            for (j, slot), blk in cell.G.items():
                got = data[f"{j}_{slot}"]
                assert np.linalg.norm(got - blk) <= 1e-11 * np.linalg.norm(blk)
    # the full factor set reloads without offline arithmetic
    back = load_offline(tmp_path, key, prob.grid, prob.partition)
    F0, F1 = layers.factors, back.factors
    for a, b in zip(F0.layers, F1.layers):
        for ca, cb in zip(a.cells, b.cells):
            assert torch.equal(ca.sinv, cb.sinv) and torch.equal(ca.green, cb.green)
            assert np.array_equal(ca.lz, cb.lz)
    assert back.backend == layers.backend and back.inner_ktol == layers.inner_ktol
    other = small_problem(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0, seed=0)
    with pytest.raises(ValueError):
        load_offline(tmp_path, key, other.grid, other.partition)
    # same grid and partition, another frequency or velocity model: rejected
    with pytest.raises(ValueError, match="omega"):
        load_offline(tmp_path, key, prob.grid, prob.partition, omega=prob.pml.omega * 1.5)
    from paper_1510_01831_b200.discretization import VelocityModel

    slower = VelocityModel(prob.grid, prob.model.c * 0.9)
    with pytest.raises(ValueError, match="another model"):
        load_offline(tmp_path, key, prob.grid, prob.partition, model=slower)
    ok = load_offline(tmp_path, key, prob.grid, prob.partition, model=prob.model, omega=prob.pml.omega)
    assert ok.factors.omega == prob.pml.omega
    # the factor file holds tensors and plain values only: it loads without unpickling code
    torch.load(tmp_path / f"factors_{key}.pt", weights_only=True)


@pytest.mark.gpu
def test_reloaded_offline_stage_solves_identically(tmp_path):
    from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers

    prob = _prob()
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc)
    dump_offline(layers, tmp_path, "k")
    back = load_offline(tmp_path, "k", prob.grid, prob.partition, device="cuda")
    f = prob.rhs([1])[0]
    cfg = KrylovConfig(ktol=1e-9)
    a = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers).solve(f, cfg)
    b = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=back).solve(f, cfg)
    assert np.array_equal(a.u, b.u) and a.iterations == b.iterations
