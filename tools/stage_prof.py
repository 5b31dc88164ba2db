"""Per-stage / per-kernel-class device time of one warm online solve (PT_STAGE_PROF breakdown).

    PT_STAGE_PROF=1 python tools/stage_prof.py --config cfg5 --nrhs 64 1

For each requested source count: one warm-up solve, one timed solve (device ms), then one profiled solve
(CUDA events around every launch; the library prints the per (stage, class) table to stderr).
"""
import argparse
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, _abi, build_nested_layers  # noqa: E402
from paper_1510_01831_b200.configs import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("nrhs", type=int, nargs="*", default=[64, 1])
ap.add_argument("--no-prof", action="store_true")
args = ap.parse_args()
prob = make_config(args.config)
t0 = time.time()
layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc,
                             inner_ktol=prob.inner_ktol, device="cuda")
solver = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
print(f"offline {time.time() - t0:.1f}s", flush=True)
cfg = KrylovConfig(ktol=prob.ktol, max_iter=prob.max_iter)
L = _abi.lib()
for R in args.nrhs:
    idx = [i % len(prob.sources) for i in range(R)]
    F = torch.from_numpy(prob.rhs(idx)).cuda()
    U = torch.empty_like(F)
    solver.solve_device(F.data_ptr(), U.data_ptr(), R, cfg)
    torch.cuda.synchronize()
    res = solver.solve_device(F.data_ptr(), U.data_ptr(), R, cfg)
    st = solver.last_stats
    print(json.dumps(dict(config=args.config, nrhs=R, device_ms=st["device_ms"],
                          its=sorted({r.iterations for r in res}), layer_solves=st["layer_solves"],
                          inner_iterations=st["inner_iterations"], touches=st["touches"],
                          launches=st["launches"])), flush=True)
    if not args.no_prof:
        L.pt_set_profiling(solver.ctx.handle, 1)
        solver.solve_device(F.data_ptr(), U.data_ptr(), R, cfg)
        L.pt_set_profiling(solver.ctx.handle, 0)
        st = solver.last_stats
        print(json.dumps(dict(nrhs=R, profiled_ms=st["device_ms"], class_ms=list(st["class_ms"]))), flush=True)
    del F, U
    torch.cuda.empty_cache()
solver.close()
