import cProfile, pstats, sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers
from paper_1510_01831_b200.configs import make_config
prob = make_config("cfg2")
layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc, device="cuda")
s = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
Fp = torch.from_numpy(prob.rhs()).pin_memory(); Up = torch.empty_like(Fp).pin_memory()
cfg = KrylovConfig(ktol=1e-9)
for _ in range(3): s.solve_many(Fp.numpy(), cfg, out=Up.numpy())
t = time.perf_counter()
for _ in range(20): s.solve_many(Fp.numpy(), cfg, out=Up.numpy())
print("e2e ms per call", (time.perf_counter() - t) / 20 * 1e3, "device ms", s.last_stats["device_ms"])
pr = cProfile.Profile(); pr.enable()
for _ in range(10): s.solve_many(Fp.numpy(), cfg, out=Up.numpy())
pr.disable(); pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
