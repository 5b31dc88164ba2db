"""GPU parity of every execution path of a sample-only layer solve (subprocess per switch set: the
library reads the switches once per process).

Default: pass-0 product + cooperative dense inner GMRES + sampled trace response.  The switches select
the direct paths that the restructuring replaces: K1 passes (PT_NO_Q0, PT_NO_GSMP), the
item-program inner GMRES (PT_NO_DENSE), the cluster dense inner GMRES (PT_NO_COOP), the fused
cooperative stage (PT_FUSE), and RECON's own first cell-solve pass instead of the saved Newton tables
plus the pass-0 product (PT_NO_REUSE).  Each must reproduce the live-reference fixture with the same iteration
counts and Green-block touches.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)

_CHILD = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, %(repo)r)
from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers
from tests.golden_cases import GOLDEN
make, si, nested = GOLDEN[%(name)r]
prob = make()
g = np.load(os.path.join(%(here)r, "golden", %(name)r + ".npz"))
layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc,
                             inner_ktol=prob.inner_ktol)
dev = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers)
res = dev.solve(prob.rhs([si])[0], KrylovConfig(ktol=float(g["ktol"]), max_iter=200))
d = int(g["decim"])
err = float(np.linalg.norm(res.u[::d, ::d] - g["u"]) / np.linalg.norm(g["u"]))
want = np.bincount(g["inner_iterations"].astype(int), minlength=64)
hist_ok = bool(np.array_equal(dev.last_stats["inner_hist"][: len(want)], want[:64]))
print(json.dumps(dict(err=err, its=res.iterations, want_its=float(g["iterations"]), hist_ok=hist_ok,
                      touches=dev.last_stats["touches"], want_touches=int(g["touches"]))))
"""

SWITCHES = {
    "default": {},
    "k1-passes": {"PT_NO_Q0": "1", "PT_NO_GSMP": "1"},
    "item-programs": {"PT_NO_DENSE": "1"},
    "item-programs-v1": {"PT_NO_DENSE": "1", "PT_ITEMS_V1": "1"},
    "cluster-dense": {"PT_NO_COOP": "1"},
    "cluster-items": {"PT_NO_DENSE": "1", "PT_NO_COOP": "1"},
    "separate-combine": {"PT_NO_FUSE_COMB": "1"},
    "inner-gather": {"PT_NO_RHS_OUT": "1"},
    "no-sstep": {"PT_NO_SSTEP": "1"},
    "pass0-segments": {"PT_P0_SEG": "1"},
    "items-tile-prefetch": {"PT_NO_DENSE": "1", "PT_ITEMS_V1": "1", "PT_TPREFETCH": "1"},
    "fused-glue": {"PT_FUSE_GLUE": "1"},
    "fused-stage": {"PT_FUSE": "1"},
    "recon-k1": {"PT_NO_REUSE": "1"},
    # the many-RHS streaming GEMM of the pass-0 product and the sampled response for every column count
    "stage-gemm": {"PT_SGEMM_MIN": "1"},
    "stage-gemm-items": {"PT_SGEMM_MIN": "1", "PT_NO_DENSE": "1"},
    # the round-1 small-N kernels of both products (the sampled response runs on the GEMM by default)
    "small-n-kernels": {"PT_NO_SGEMM": "1"},
}


@pytest.mark.parametrize("name", ["small_b", "small_c", "cfg1"])
@pytest.mark.parametrize("switch", list(SWITCHES))
def test_execution_paths_match_reference_fixture(name, switch):
    env = dict(os.environ, **SWITCHES[switch])
    code = _CHILD % dict(repo=REPO, here=HERE, name=name)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["err"] <= 1e-8, r
    assert r["its"] == r["want_its"], r
    assert r["hist_ok"], r
    assert r["touches"] == r["want_touches"], r
