"""One K1 launch on one cfg2 cell (dense test path), for ncu."""
import os, sys
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
x = solver.cell_solve(1, 1, b)
x = solver.cell_solve(1, 1, b)
print("ok", np.abs(x).max())
