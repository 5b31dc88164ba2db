#!/usr/bin/env python
"""Benchmark: online stage of the nested polarized-traces solver on one B200 per rank.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

A step is one online solve of the config's whole source set (config 2 =
BASELINE.json configs[1]: 400x400 Gaussian lens, L=8, Lc=4, 16 point sources),
batched through ``pt_solve_device`` with sources and wavefields resident in HBM
(``value``), and through the public API with pinned host buffers, H2D/D2H
inside the timed region (``e2e``).  One process per GPU (torchrun for N>1);
each rank solves its own copy of the source set (weak scaling, no collective
on the data path); the step time is the max over ranks.

Roofline: the dominant kernel is K1 (cell solves).  Its algorithmic work is
SURVEY.md 8(d)'s ``32 wz_c w_c^2`` bytes of Schur inverse per cell solve per
RHS (flops = bytes/2).  With 16 RHS batched per stage the factor bytes are
shared across RHS, so the bound is the FP64 pipe: achieved FLOP/s of K1 over
its summed CUDA-event time in the timed region, against the measured FP64
peak (profiles/fp64_peak.json, measured on the B200 by tools/fp64_peak.cu).

``--impl reference`` times the CPU oracle port (oracle/, the reference's
algorithm on SuperLU + BLAS) on the host cores: offline once, then each step
solves a sample of the sources in forked worker processes (one per core).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

if "reference" in sys.argv:  # the CPU arm: one BLAS thread per worker process (set before numpy loads)
    for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(_v, "1")

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "online solves/s (complex128 nested polarized-traces solve, whole source set)"
UNIT = "solves/s"


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def _peaks():
    out = {"hbm_gbs": 6536.4, "hbm_src": "fallback"}
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
        out["hbm_gbs"] = float(mp["hbm_gbs"])
        out["hbm_src"] = "measured (MEASURED_PEAKS.json)"
        out["sm_max_mhz"] = float(mp.get("sm_max_mhz", 1965.0))
    except Exception:
        pass
    try:
        with open(os.path.join(REPO, "profiles", "fp64_peak.json")) as fh:
            fp = json.load(fh)
        out["fp64_tflops"] = float(max(fp["dfma_tflops"], fp["dmma_tflops"]))
        out["fp64_src"] = "measured on B200 (profiles/fp64_peak.json)"
    except Exception:
        out["fp64_tflops"] = 40.0
        out["fp64_src"] = "nominal B200 FP64 (no measurement found)"
    return out


def _inner_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture, or None."""
    try:
        with open(os.path.join(REPO, "profiles", "r01_inner_traffic.json")) as fh:
            return float(json.load(fh)["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 10 ms during the timed region through NVML
    (in-process, so even a region of a few tens of ms gets samples); nvidia-smi -lms 200 if NVML is absent."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clock-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self._sample()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _sample(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.samples.append((float(sm), float(mx), int(rs)))

    def _poll(self):
        while not self.stop.wait(0.01):
            try:
                self._sample()
            except Exception:
                return

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml is not None:
            try:
                self._sample()  # the region's last moment
            except Exception:
                pass
            self.stop.set()
            self.t.join(timeout=1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for s_, m_, bits in self.samples:
            sm.append(s_)
            mx = max(mx, m_)
            for nm, bit in self.BITS.items():
                if bits & bit:
                    reasons.add(nm)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml (10 ms)" if self.nvml is not None else "nvidia-smi (200 ms)"}


def _cpu_baseline_sample(cfg_name, n_src, threads):
    """Run the oracle on a bounded sample in a subprocess with `threads` BLAS threads."""
    code = f"""
import sys, time, json
sys.path.insert(0, {REPO!r})
from oracle.polartraces_oracle import OracleSolver
from paper_1510_01831_b200.configs import make_config
prob = make_config({cfg_name!r})
t0 = time.time(); s = OracleSolver.from_problem(prob); t1 = time.time()
F = prob.rhs(list(range({n_src})))
t2 = time.time()
for f in F:
    s.solve(f, ktol=prob.ktol, max_iter=prob.max_iter)
t3 = time.time()
print(json.dumps({{"offline_s": t1 - t0, "solve_s": t3 - t2}}))
"""
    env = dict(os.environ, OPENBLAS_NUM_THREADS=str(threads), OMP_NUM_THREADS=str(threads),
               MKL_NUM_THREADS=str(threads))
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         timeout=900)
    if res.returncode != 0:
        raise RuntimeError(res.stderr[-2000:])
    return json.loads(res.stdout.strip().splitlines()[-1])


# ----------------------------------------------------------------------------- reference arm

_REF = {}


def _ref_init():
    # one BLAS thread per worker process: numpy was initialised before the fork
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def _ref_worker(idx):
    s, F, prob = _REF["s"], _REF["F"], _REF["prob"]
    r = s.solve(F[idx], ktol=prob.ktol, max_iter=prob.max_iter)
    return r.iterations


def run_reference(args):
    rank, local, world = _env_rank()
    if rank != 0:
        return 0
    import multiprocessing as mp

    from oracle.polartraces_oracle import OracleSolver
    from paper_1510_01831_b200.configs import make_config

    prob = make_config(args.config)
    t0 = time.time()
    s = OracleSolver.from_problem(prob)
    offline = time.time() - t0
    cores = os.cpu_count() or 1
    n_sample = min(len(prob.sources), cores)
    _REF.update(s=s, F=prob.rhs(list(range(len(prob.sources)))), prob=prob)
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(n_sample, initializer=_ref_init) as pool:
        for step in range(args.warmup + args.steps):
            t = time.time()
            its = pool.map(_ref_worker, [(step * n_sample + i) % len(prob.sources) for i in range(n_sample)])
            dt = time.time() - t
            if step >= args.warmup:
                times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = n_sample / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": _config(args, prob),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": n_sample, "kind": "port",
                         "sample": f"{n_sample} of the {len(prob.sources)} {args.config} sources per step, "
                                   f"one forked oracle process per core (OPENBLAS_NUM_THREADS=1); "
                                   f"offline {offline:.1f}s untimed; outer its {sorted(set(its))}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(args, prob):
    g = prob.grid
    R = len(prob.sources) if getattr(args, "nrhs", 0) <= 0 else min(args.nrhs, len(prob.sources))
    return {"workload": f"{args.config}: {g.nx}x{g.nz} interior + {g.npml}-pt PML, L={prob.partition.L}, "
                        f"Lc={prob.Lc}, {R} point sources batched per step",
            "unknowns": g.nx * g.nz, "nrhs": R, "ktol": prob.ktol,
            "inner_ktol": prob.inner_ktol, "preconditioner": "gs",
            "inner_backend": getattr(args, "backend", "pt"),
            "l2": "factor working set (Schur inverses) larger than the 126 MB L2; no explicit flush",
            "parallelism": f"rhs-replica x{args.gpus}"}


# ----------------------------------------------------------------------------- our arm


def run_ours(args):
    import torch

    rank, local, world = _env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers
    from paper_1510_01831_b200 import _abi
    from paper_1510_01831_b200.configs import make_config

    prob = make_config(args.config)
    t0 = time.time()
    layers = build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition, Lc=prob.Lc,
                                 inner_ktol=prob.inner_ktol, device=f"cuda:{local}", backend=args.backend)
    solver = PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition, layers=layers,
                                   device=local)
    offline_s = time.time() - t0
    R = len(prob.sources) if args.nrhs <= 0 else min(args.nrhs, len(prob.sources))
    Fh = prob.rhs(list(range(R)))
    F = torch.from_numpy(Fh).to(f"cuda:{local}")
    U = torch.empty_like(F)
    cfg = KrylovConfig(ktol=prob.ktol, max_iter=prob.max_iter)
    stream = torch.cuda.current_stream()
    L = _abi.lib()
    L.pt_set_stream(solver.ctx.handle, C_void(stream.cuda_stream))

    def step():
        return solver.solve_device(F.data_ptr(), U.data_ptr(), R, cfg)

    for _ in range(max(args.warmup, 3 if args.warmup >= 3 else args.warmup)):
        res = step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = 0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()  # `ncu --profile-from-start off` sees the timed region only
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            res = step()
            launches += solver.last_stats["launches"]
        e1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # per-launch-class device time from a separate profiled pass (CUDA events around every launch add
    # overhead, so they stay out of the timed region); drives the roofline and the shares
    L.pt_set_profiling(solver.ctx.handle, 1)
    prof_steps = 2
    cls_ms = np.zeros(5)
    k1_bytes = dense_flops = prof_ms = 0.0
    for _ in range(prof_steps):
        step()
        st = solver.last_stats
        cls_ms += st["class_ms"]
        k1_bytes += st["k1_bytes"]
        dense_flops += st["dense_flops"]
        prof_ms += st["device_ms"]
    L.pt_set_profiling(solver.ctx.handle, 0)
    value = R * world / (ms / 1e3)

    # end to end through the public API: pinned host f in, host u out, copies inside the timed region
    Fp = torch.from_numpy(Fh).pin_memory()
    Up = torch.empty_like(Fp).pin_memory()
    L.pt_set_stream(solver.ctx.handle, None)
    solver.solve_many(Fp.numpy(), cfg, out=Up.numpy())
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t = time.perf_counter()
    for _ in range(args.steps):
        out = solver.solve_many(Fp.numpy(), cfg, out=Up.numpy())
    e2e_ms = 1e3 * (time.perf_counter() - t) / args.steps
    if dist:
        tt = torch.tensor([e2e_ms], device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e = R * world / (e2e_ms / 1e3)
    nbytes = int(Fh.nbytes)

    # parity spot check of this run's wavefield against the committed reference fixture
    parity = None
    gpath = os.path.join(REPO, "tests", "golden",
                         f"{args.config}{'' if args.backend == 'pt' else '_' + args.backend}.npz")
    if os.path.exists(gpath):
        g = np.load(gpath)
        d = int(g["decim"])
        u0 = U[0].cpu().numpy()[::d, ::d]
        parity = float(np.linalg.norm(u0 - g["u"]) / np.linalg.norm(g["u"]))

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    peaks = _peaks()
    names = ["k1_cell_solve", "inner_gmres", "glue", "green_samples", "pass0_product"]
    k1_tf = (k1_bytes / 2.0) / (cls_ms[0] * 1e-3) / 1e12 if cls_ms[0] > 0 else 0.0
    inner_tf = dense_flops / (cls_ms[1] * 1e-3) / 1e12 if cls_ms[1] > 0 else 0.0
    dom = int(np.argmax(cls_ms[:2]))
    achieved_tf = inner_tf if dom == 1 else k1_tf
    its = sorted({r.iterations for r in res})
    # SURVEY 8(d) algorithmic work of the reference's online solve for this batch: every layer solve is
    # 2 cell solves per cell, each reading its Schur factors twice (2 x 32 wz_c w_c^2 B), plus 16 B per
    # inner Green-block touch; layer solves and touches are this step's own counts (identical to the
    # reference's), per-layer bytes averaged over the layers (their heights differ by at most one row)
    st_last = solver.last_stats
    F_ = layers.factors
    per_layer = [sum(64.0 * cf.wzc * cf.w * cf.w for cf in lf.cells) for lf in F_.layers]
    alg_bytes = st_last["layer_solves"] * float(np.mean(per_layer)) + 16.0 * st_last["touches"]
    alg_gbs = alg_bytes / (ms * 1e-3) / 1e9
    alg_tf = alg_bytes / 2.0 / (ms * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded config generator, SURVEY 8(d))",
        "config": _config(args, prob),
        "munknowns_rhs_per_s": value * prob.grid.nx * prob.grid.nz / 1e6,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes},
        "gpu_launches": int(launches),
        "roofline": {
            "kernel": names[dom], "bound": "tensor", "unit": "TFLOP/s",
            "achieved": achieved_tf, "peak": peaks["fp64_tflops"],
            "frac": achieved_tf / peaks["fp64_tflops"], "traffic": _inner_traffic(),
            "traffic_src": "profiles/r01_inner_traffic.json: ncu dram__bytes_read+write per inner launch, averaged "
                           "over the 57 inner launches of one solve (bytes per launch)",
            "peak_src": peaks["fp64_src"],
            "algorithmic": ("inner: 8 n^2 flops per instance per dense product (n = 4 (Lc-1) w), products = "
                            "inner iterations + inner solves; K1: 32*wz_c*w_c^2 B per cell solve per RHS "
                            "(SURVEY 8(d)), flops = bytes/2"),
            "class_share_of_step": {nm: float(c / prof_steps / ms) for nm, c in zip(names, cls_ms)},
            "k1_tflops": k1_tf, "inner_dense_tflops": inner_tf,
            "profiled_ms_per_step": prof_ms / prof_steps,
        },
        "solve_roofline": {
            "formula": "SURVEY 8(d): sum_l N_l sum_c 2*32*wz_c*w_c^2 B + 16 B per inner touch; flops = bytes/2",
            "bytes_per_rhs": alg_bytes / R, "achieved_gbs": alg_gbs, "hbm_peak_gbs": peaks["hbm_gbs"],
            "hbm_frac": alg_gbs / peaks["hbm_gbs"], "achieved_tflops": alg_tf,
            "fp64_peak_tflops": peaks["fp64_tflops"], "fp64_frac": alg_tf / peaks["fp64_tflops"],
            "regime": "1 RHS: HBM bound" if R == 1 else f"{R} RHS per step: FP64 tensor bound",
        },
        "clocks": clk.summary(),
        "outer_iterations": its,
        "parity_vs_reference_fixture": parity,
        "offline_s": offline_s,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            cb = _cpu_baseline_sample(args.config, 1, 1)
            line["cpu_baseline"] = {"value": 1.0 / cb["solve_s"], "unit": UNIT, "cores": 1, "kind": "port",
                                    "sample": f"1 {args.config} source solved by the oracle port "
                                              f"(single process, OPENBLAS_NUM_THREADS=1, offline "
                                              f"{cb['offline_s']:.1f}s untimed)"}
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "port",
                                    "sample": f"failed: {exc!s:.200}"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def C_void(x):
    import ctypes

    return ctypes.c_void_p(x)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nrhs", type=int, default=0, help="solve the config's first N sources (0 = all)")
    ap.add_argument("--backend", default="pt", choices=["pt", "lu"],
                    help="inner backend (build_nested_layers backend=; the benchmark line uses 'pt')")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
