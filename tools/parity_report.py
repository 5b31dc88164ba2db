"""Print parity numbers of the B200 path vs the golden fixtures (diagnostic)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers
from tests.golden_cases import GOLDEN

HERE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")
for name in sys.argv[1:] or list(GOLDEN):
    make, si, nested = GOLDEN[name]
    prob = make()
    g = np.load(os.path.join(HERE, "golden", f"{name}.npz"))
    t0 = time.time()
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition,
                                 Lc=prob.Lc if nested else 1, device="cuda")
    dev = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
    t1 = time.time()
    f = prob.rhs([si])[0]
    for rep in range(3):
        t2 = time.time()
        res = dev.solve(f, KrylovConfig(ktol=float(g["ktol"])))
        t3 = time.time()
    d = int(g["decim"])
    err = np.linalg.norm(res.u[::d, ::d] - g["u"]) / np.linalg.norm(g["u"])
    st = dev.last_stats
    print(f"{name}: relL2={err:.3e} its={res.iterations} (ref {float(g['iterations'])}) "
          f"res={np.array(res.residuals)} ref={g['residuals']} relres={res.relative_residual:.4e} "
          f"(ref {float(g['relres']):.4e}) touches={st['touches']} (ref {int(g['touches'])}) "
          f"ls={st['layer_solves']} inner={st['inner_iterations']} offline={t1-t0:.2f}s "
          f"solve={1e3*(t3-t2):.2f}ms dev={st['device_ms']:.2f}ms", flush=True)
