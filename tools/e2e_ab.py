import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ctypes as C
from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers, _abi
from paper_1510_01831_b200.configs import make_config
prob = make_config("cfg2")
layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc, device="cuda")
s = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
Fp = torch.from_numpy(prob.rhs()).pin_memory(); Up = torch.empty_like(Fp).pin_memory()
cfg = KrylovConfig(ktol=1e-9)
for _ in range(5): s.solve_many(Fp.numpy(), cfg, out=Up.numpy())
t = time.perf_counter()
for _ in range(20): s.solve_many(Fp.numpy(), cfg, out=Up.numpy())
print("solve_many ms", (time.perf_counter() - t) / 20 * 1e3)
# raw pt_solve without trace/polarized outputs
R = 16
kc = _abi.PtKrylov(1e-9, 200, 0, 1e-6, 200, 0, 0)
st = _abi.PtStats()
F = Fp.numpy(); U = Up.numpy()
L = _abi.lib()
for _ in range(3): L.pt_solve(s.ctx.handle, _abi.dptr(F.view(np.float64)), R, C.byref(kc), _abi.dptr(U.view(np.float64)), C.byref(st))
t = time.perf_counter()
for _ in range(20): L.pt_solve(s.ctx.handle, _abi.dptr(F.view(np.float64)), R, C.byref(kc), _abi.dptr(U.view(np.float64)), C.byref(st))
print("pt_solve (no stats) ms", (time.perf_counter() - t) / 20 * 1e3)
