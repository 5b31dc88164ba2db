"""One warm cfg2 online solve bracketed by cudaProfilerStart/Stop (for ncu --profile-from-start off).

    python tools/profile_solve.py [--config cfg2] [--nrhs 16] [--label]
With --label, prints the per-launch class/time table from the library's own CUDA events.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers  # noqa: E402
from paper_1510_01831_b200.configs import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--nrhs", type=int, default=16)
args = ap.parse_args()
prob = make_config(args.config)
layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc, device="cuda")
solver = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
idx = [i % len(prob.sources) for i in range(args.nrhs)]
F = torch.from_numpy(prob.rhs(idx)).cuda()
U = torch.empty_like(F)
cfg = KrylovConfig(ktol=prob.ktol)
for _ in range(2):
    solver.solve_device(F.data_ptr(), U.data_ptr(), args.nrhs, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = solver.solve_device(F.data_ptr(), U.data_ptr(), args.nrhs, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("its", sorted({r.iterations for r in res}), "device_ms", solver.last_stats["device_ms"],
      "launches", solver.last_stats["launches"])
