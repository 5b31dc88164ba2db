"""Time K1 alone (dense cell-solve test path) on a cfg2 cell under PT_K1_DBG switches."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_01831_b200 import PolarizedTracesSolver, build_nested_layers
from paper_1510_01831_b200.configs import make_config
prob = make_config("cfg2")
layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc, device="cuda")
solver = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
cf = layers.factors.layers[1].cells[1]
nc = int(os.environ.get("PT_K1_NC", "8"))
b = np.random.default_rng(0).standard_normal((nc, cf.wzc, cf.w)) + 0j
for _ in range(3):
    x = solver.cell_solve(1, 1, b)
t = time.perf_counter()
for _ in range(20):
    x = solver.cell_solve(1, 1, b)
dt = (time.perf_counter() - t) / 20
print(f"nc={nc} dbg={os.environ.get('PT_K1_DBG', '0')}: {dt*1e6:.0f} us per call (incl. H2D/D2H), "
      f"{dt*1e6/61:.2f} us per step upper bound")
