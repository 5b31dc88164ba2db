"""Offline artifacts built from the LIVE reference's own layer objects (build container only).

    python tests/golden/make_refobj.py

``PolarizedTracesSolver(layers=<reference build_nested_layers output>)`` reads the reference's assembled
operators and uploads its GreenBlockSet matrices (solver.from_reference_layers).  The reference is not on the
GPU box, so the factors produced from its objects for the small_b problem are dumped here
(artifacts.dump_offline) and the GPU test solves with them (tests/test_gpu_parity.py).
"""

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import polartraces as rpt  # noqa: E402

from paper_1510_01831_b200.artifacts import dump_offline  # noqa: E402
from paper_1510_01831_b200.solver import from_reference_layers  # noqa: E402
from paper_1510_01831_b200.configs import small_problem  # noqa: E402
from tests.golden_cases import REFOBJ_CASE  # noqa: E402

prob = small_problem(**REFOBJ_CASE)
g = prob.grid
grid = rpt.Grid(g.nx, g.nz, g.h, g.npml)
model = rpt.VelocityModel(grid, prob.model.c)
pml = rpt.PmlProfile(g.npml, g.h, prob.pml.C, prob.pml.omega)
part = rpt.LayerPartition(tuple(prob.partition.extents))
ref_layers = rpt.build_nested_layers(grid, model, pml, part, Lc=prob.Lc, inner_ktol=prob.inner_ktol)
layers = from_reference_layers(ref_layers, prob.grid, prob.model, prob.pml, prob.partition, inner_dense=False)
out = os.path.join(HERE, "refobj")
shutil.rmtree(out, ignore_errors=True)
dump_offline(layers, out, "refobj", model=prob.model, grid=prob.grid, omega=prob.pml.omega, partition=prob.partition)
for fn in os.listdir(out):  # only the factor file and its manifest are needed by the test
    if fn.startswith("green_"):
        os.remove(os.path.join(out, fn))
print(sorted(os.listdir(out)))

# ---- the same from PLR-compressed reference layers (plr_threshold below the cell width, so every Green block is
# a PlrMatrix): factors built from the reference objects (blocks expanded by GreenBlockSet.dense) plus the
# reference's own solves with those compressed layers, which the device must reproduce
import numpy as np  # noqa: E402

from tests.golden_cases import REFOBJ_PLR  # noqa: E402

plr_layers = rpt.build_nested_layers(grid, model, pml, part, Lc=prob.Lc, inner_ktol=prob.inner_ktol, **REFOBJ_PLR)
assert all(isinstance(m, rpt.plr.PlrMatrix) for lay in plr_layers for bs in lay.blocksets for m in bs.blocks.values())
layers = from_reference_layers(plr_layers, prob.grid, prob.model, prob.pml, prob.partition, inner_dense=False)
out = os.path.join(HERE, "refobj_plr")
shutil.rmtree(out, ignore_errors=True)
dump_offline(layers, out, "refobj_plr", model=prob.model, grid=prob.grid, omega=prob.pml.omega,
             partition=prob.partition)
for fn in os.listdir(out):
    if fn.startswith("green_"):
        os.remove(os.path.join(out, fn))
ref = rpt.PolarizedTracesSolver(grid, model, pml, part, layers=plr_layers)
res = [ref.solve(f, rpt.KrylovConfig(ktol=1e-9)) for f in prob.rhs()]
np.savez_compressed(os.path.join(HERE, "refobj_plr.npz"), u=np.stack([r.u for r in res]),
                    iterations=np.array([r.iterations for r in res]),
                    relres=np.array([r.relative_residual for r in res]))
print(sorted(os.listdir(out)), [r.iterations for r in res])
