"""Generate golden fixtures by running the LIVE reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (``/root/reference/pkg/src/polartraces``) is importable here but
does not exist on the GPU box, so its outputs are committed as small ``.npz``
fixtures.  Inputs come from ``paper_1510_01831_b200.configs`` so both sides see
identical problems.  Recorded per case: wavefield (full for the small cases,
every 4th node for config 1), outer GMRES iteration count and residual
history, true relative residual, the inner ``TouchCounter`` total, and the
per-layer-solve inner GMRES iteration counts (via a wrapper around
``nested.krylov.gmres``).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import polartraces as pt  # noqa: E402
from polartraces import krylov as ref_krylov  # noqa: E402
from polartraces import nested as ref_nested  # noqa: E402

from paper_1510_01831_b200.configs import make_config, small_problem  # noqa: E402

_INNER = []
_orig_gmres = ref_krylov.gmres


_STATE = {"in_solve": False, "depth": 0}
_orig_solve = ref_krylov.solve


def _counting_gmres(*a, **kw):
    # record every gmres call except the outer one (the call krylov.solve
    # makes at depth 1, sie.py:419); inner calls come from nested.py:147
    _STATE["depth"] += 1
    try:
        res = _orig_gmres(*a, **kw)
    finally:
        _STATE["depth"] -= 1
    if not (_STATE["in_solve"] and _STATE["depth"] == 0):
        _INNER.append(res.iterations)
    return res


def _outer_solve(*a, **kw):
    _STATE["in_solve"] = True
    try:
        return _orig_solve(*a, **kw)
    finally:
        _STATE["in_solve"] = False


_orig_bicgstab = ref_krylov.bicgstab


def _outer_bicgstab(*a, **kw):
    # the outer BiCGstab: inner gmres calls made under it are one level down
    _STATE["depth"] += 1
    try:
        return _orig_bicgstab(*a, **kw)
    finally:
        _STATE["depth"] -= 1


ref_krylov.gmres = _counting_gmres
ref_krylov.solve = _outer_solve
ref_krylov.bicgstab = _outer_bicgstab


def ref_solver(prob, nested=True, backend="pt", assembled=False):
    g = prob.grid
    grid = pt.Grid(g.nx, g.nz, g.h, g.npml)
    model = pt.VelocityModel(grid, prob.model.c)
    pml = pt.PmlProfile(g.npml, g.h, prob.pml.C, prob.pml.omega)
    part = pt.LayerPartition(tuple(prob.partition.extents))
    layers = None
    if nested:
        layers = pt.build_nested_layers(grid, model, pml, part, Lc=prob.Lc, backend=backend,
                                        inner_ktol=prob.inner_ktol, assembled_boundary=assembled)
    return pt.PolarizedTracesSolver(grid, model, pml, part, layers=layers)


def run_case(prob, src_idx, nested=True, ktol=1e-9, full_u=True, decim=1, method="gmres", backend="pt",
             assembled=False, solver=None, traces=False, trace_decim=1):
    t0 = time.time()
    s = solver if solver is not None else ref_solver(prob, nested, backend, assembled)
    t1 = time.time()
    f = prob.rhs([src_idx])[0]
    _INNER.clear()
    for lay in s.layers:
        if hasattr(lay, "counter"):
            lay.counter.reset()
    res = s.solve(f, pt.KrylovConfig(ktol=ktol, max_iter=200, method=method))
    t2 = time.time()
    touches = sum(lay.counter.total for lay in s.layers if hasattr(lay, "counter"))
    u = res.u if full_u else res.u[::decim, ::decim]
    out = dict(
        u=u,
        decim=decim,
        unorm=np.linalg.norm(res.u),
        iterations=res.iterations,
        residuals=np.array(res.residuals),
        relres=res.relative_residual,
        touches=touches,
        inner_iterations=np.array(_INNER, dtype=float),
        source=np.array(prob.sources[src_idx]),
        ktol=ktol,
        nested=nested,
        method=method,
        backend=backend,
        assembled=assembled,
        offline_s=t1 - t0,
        online_s=t2 - t1,
        src_idx=src_idx,
    )
    if traces and res.traces is not None:  # SolveResult.traces (sie.py:426-427), (nI, 2, wx)
        out["traces"] = res.traces.data[:, :, ::trace_decim]
        out["trace_decim"] = trace_decim
    print(f"{prob.name} src{src_idx} nested={nested}: its={res.iterations} "
          f"res={res.residuals} relres={res.relative_residual:.3e} touches={touches} "
          f"inner={len(_INNER)} offline={t1 - t0:.2f}s online={t2 - t1:.2f}s")
    return out


BIG = {"cfg1": 4, "cfg2": 8, "cfg3": 8, "cfg4": 8, "cfg5": 12}  # wavefield decimation


_FORK = {}


def _fork_solve(job):
    prob, s, name, decim, tdec = _FORK["prob"], _FORK["s"], _FORK["name"], _FORK["decim"], _FORK["tdec"]
    out = run_case(prob, job, full_u=decim == 1, decim=decim, solver=s, traces=True, trace_decim=tdec)
    out["offline_s"] = _FORK["offline_s"]
    np.savez_compressed(os.path.join(HERE, f"{name}_s{job}.npz"), **out)
    return job


def sources(name, idx, decim=None, tdec=1):
    """Per-source fixtures ``<name>_s<k>.npz`` of one config: the reference is built once (offline), then
    the sources are solved in forked processes (the factors are shared copy-on-write and read-only)."""
    import multiprocessing as mp

    prob = make_config(name)
    t0 = time.time()
    s = ref_solver(prob)
    _FORK.update(prob=prob, s=s, name=name, decim=BIG[name] if decim is None else decim, tdec=tdec,
                 offline_s=time.time() - t0)
    print(f"{name}: offline {time.time() - t0:.1f}s; solving sources {idx}", flush=True)
    with mp.get_context("fork").Pool(len(idx)) as pool:
        for k in pool.imap_unordered(_fork_solve, idx):
            print(f"{name} source {k} done", flush=True)


def main(argv):
    # ``make_golden.py cfg3 [cfg4 ...]`` regenerates only the named large configs
    # (cfg3 takes minutes, cfg4 tens of minutes, cfg5 hours on the reference)
    if argv == ["assembled"]:  # the factored boundary pipeline (nested.py:355-486, Eq. 4.3)
        for name, prob, si, decim, backend in (
                ("small_b", small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 1, 1, "pt"),
                ("small_c", small_problem(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7), 0, 1, "lu"),
                ("cfg1", make_config("cfg1"), 0, 4, "pt")):
            out = run_case(prob, si, full_u=decim == 1, decim=decim, backend=backend, assembled=True)
            np.savez_compressed(os.path.join(HERE, f"{name}_asm.npz"), **out)
        return
    if argv == ["lu"]:  # the direct inner backend (nested.py:156-269)
        for name, prob, si, decim in (
                ("small_b", small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 1, 1),
                ("small_c", small_problem(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7), 0, 1),
                ("cfg1", make_config("cfg1"), 0, 4), ("cfg2", make_config("cfg2"), 0, 8)):
            out = run_case(prob, si, full_u=decim == 1, decim=decim, backend="lu")
            np.savez_compressed(os.path.join(HERE, f"{name}_lu.npz"), **out)
        return
    if argv == ["bicgstab"]:  # the outer BiCGstab path (krylov.py:138-201)
        for name, prob, decim in (("small_b", small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 1),
                                  ("cfg1", make_config("cfg1"), 4)):
            out = run_case(prob, 1 if name == "small_b" else 0, full_u=decim == 1, decim=decim,
                           method="bicgstab")
            np.savez_compressed(os.path.join(HERE, f"{name}_bicgstab.npz"), **out)
        return
    if argv and argv[0] == "sources":
        # ``make_golden.py sources cfg3 21 42 63 [--decim D] [--tdec T]``: per-source fixtures of the
        # many-RHS source sets (sie.py:392-439 solves each source independently)
        rest = argv[1:]
        opts = {}
        while "--decim" in rest or "--tdec" in rest:
            i = rest.index("--decim") if "--decim" in rest else rest.index("--tdec")
            opts[rest[i][2:]] = int(rest[i + 1])
            del rest[i:i + 2]
        sources(rest[0], [int(x) for x in rest[1:]], decim=opts.get("decim"), tdec=opts.get("tdec", 1))
        return
    if argv:
        for name in argv:
            prob = make_config(name)
            out = run_case(prob, 0, full_u=False, decim=BIG[name])
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        return
    cases = {
        "small_a": (small_problem(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0, seed=0), 0, True),
        "small_b": (small_problem(nx=48, nz=41, npml=5, L=4, Lc=3, omega=20.0, seed=3), 1, True),
        "small_c": (small_problem(nx=33, nz=30, npml=4, L=2, Lc=4, omega=11.0, seed=7), 0, True),
        "small_direct": (small_problem(nx=40, nz=36, npml=6, L=3, Lc=2, omega=14.0, seed=0), 0,
                         False),
    }
    for name, (prob, si, nested) in cases.items():
        out = run_case(prob, si, nested=nested)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    for name, decim in (("cfg1", 4), ("cfg2", 8)):
        prob = make_config(name)
        out = run_case(prob, 0, full_u=False, decim=decim)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


if __name__ == "__main__":
    main(sys.argv[1:])
