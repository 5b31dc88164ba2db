"""Solve a subset of one benchmark config's sources on the B200 and report time, iterations and parity.

    python tools/run_config.py cfg4 --sources 0 1 2 --repeat 2

Offline factors are built on the GPU (torch).  The wavefield of source 0 is compared with the committed
live-reference fixture ``tests/golden/<cfg>.npz`` when it exists (relative L2 on the fixture's decimated
grid, outer iterations, residual history, Green-block touches and the inner iteration histogram).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--sources", type=int, nargs="*", default=[0])
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--inner-dense", type=int, default=None)
    args = ap.parse_args()
    import torch

    from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers
    from paper_1510_01831_b200.configs import make_config

    prob = make_config(args.config)
    t0 = time.time()
    dense = None if args.inner_dense is None else bool(args.inner_dense)
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc,
                                 inner_ktol=prob.inner_ktol, device="cuda", inner_dense=dense)
    t1 = time.time()
    solver = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
    t2 = time.time()
    print(f"offline build {t1 - t0:.1f}s upload {t2 - t1:.1f}s; "
          f"gpu mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB (torch)", flush=True)
    F = prob.rhs(args.sources)
    cfg = KrylovConfig(ktol=prob.ktol, max_iter=prob.max_iter)
    out = {}
    for rep in range(args.repeat):
        t = time.time()
        res = solver.solve_many(F, cfg)
        dt = time.time() - t
        st = solver.last_stats
        out = dict(config=args.config, nrhs=len(args.sources), wall_s=dt, device_ms=st["device_ms"],
                   solves_per_s=len(args.sources) / (st["device_ms"] / 1e3),
                   iterations=[r.iterations for r in res], relres=[r.relative_residual for r in res],
                   layer_solves=st["layer_solves"], inner_iterations=st["inner_iterations"],
                   touches=st["touches"], launches=st["launches"])
        print(json.dumps(out), flush=True)
    g_path = os.path.join(REPO, "tests", "golden", f"{args.config}.npz")
    if 0 in args.sources and os.path.exists(g_path):
        g = np.load(g_path)
        i0 = args.sources.index(0)
        # single-source solve for the per-source counters
        r0 = solver.solve(F[i0], cfg)
        st = solver.last_stats
        d = int(g["decim"])
        err = float(np.linalg.norm(r0.u[::d, ::d] - g["u"]) / np.linalg.norm(g["u"]))
        want = np.bincount(g["inner_iterations"].astype(int), minlength=64)
        print(json.dumps(dict(
            parity_rel_l2=err, iterations=r0.iterations, ref_iterations=float(g["iterations"]),
            residuals=r0.residuals, ref_residuals=list(map(float, g["residuals"])),
            touches=st["touches"], ref_touches=int(g["touches"]),
            inner_hist_equal=bool(np.array_equal(st["inner_hist"][: len(want)], want[:64])),
            unorm=float(np.linalg.norm(r0.u)), ref_unorm=float(g["unorm"]),
            ref_online_s=float(g["online_s"]), ref_offline_s=float(g["offline_s"]))), flush=True)
    solver.close()


if __name__ == "__main__":
    main()
