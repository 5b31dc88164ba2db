"""K1 alone (usage: k1_probe.py [1x64,2x32,... [dbg,dbg]]) on the dense cell-solve test path: one cfg2 cell, `tasks` CTA pairs of nc columns each,
under PT_K1_DBG switches (1: consumers skip the data waits; 2: consumers skip the matvec).
Prints the launch time and CTA 0's per-phase clock64 totals (PT_K1_TPROF)."""
import os, subprocess, sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    from paper_1510_01831_b200 import PolarizedTracesSolver, build_nested_layers
    from paper_1510_01831_b200.configs import make_config
    prob = make_config("cfg2")
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc, device="cuda")
    solver = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
    cf = layers.factors.layers[1].cells[1]
    nrhs = int(sys.argv[2])
    b = np.random.default_rng(0).standard_normal((nrhs, cf.wzc, cf.w)) + 0j
    for _ in range(3):
        solver.cell_solve(1, 1, b)
    sys.exit(0)

cases = [(1, 64), (2, 32), (4, 16), (8, 8)]
dbgs = (0, 1, 2)
if len(sys.argv) > 1:
    cases = [tuple(int(v) for v in c.split("x")) for c in sys.argv[1].split(",")]
    dbgs = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 else (0,)
for nc, tasks in cases:
    for dbg in dbgs:
        env = dict(os.environ, PT_K1_NC=str(nc), PT_K1_DBG=str(dbg), PT_K1_TPROF="1")
        r = subprocess.run([sys.executable, __file__, "--child", str(nc * tasks)], env=env, capture_output=True, text=True)
        lines = [l for l in r.stderr.splitlines() if l.startswith("cell_solve")]
        print(lines[-1] if lines else f"nc={nc} dbg={dbg} FAILED: {r.stderr[-300:]}", flush=True)
