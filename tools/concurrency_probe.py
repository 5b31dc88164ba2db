"""Probe: two independent contexts (8 sources each) solving concurrently on two streams from two host
threads, against one context with all 16 sources.  PT_COOP_SMS caps the cooperative inner kernels' grid."""
import os, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_01831_b200 import KrylovConfig, PolarizedTracesSolver, build_nested_layers, _abi
from paper_1510_01831_b200.configs import make_config
import ctypes

prob = make_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
R = len(prob.sources)
cfg = KrylovConfig(ktol=prob.ktol)
mk = lambda: PolarizedTracesSolver(prob.grid, prob.model, prob.pml, prob.partition,
                                   layers=build_nested_layers(prob.grid, prob.model, prob.pml, prob.partition,
                                                              Lc=prob.Lc, device="cuda"))
F = torch.from_numpy(prob.rhs()).cuda()
U = torch.empty_like(F)
one = mk()
for _ in range(3):
    one.solve_device(F.data_ptr(), U.data_ptr(), R, cfg)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    one.solve_device(F.data_ptr(), U.data_ptr(), R, cfg)
torch.cuda.synchronize()
t1 = (time.perf_counter() - t) / 10
print(f"one context, {R} sources: {t1 * 1e3:.2f} ms per step", flush=True)
two = [mk(), mk()]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
h = R // 2
for k in range(2):
    _abi.lib().pt_set_stream(two[k].ctx.handle, ctypes.c_void_p(streams[k].cuda_stream))
def run(k, n):
    for _ in range(n):
        two[k].solve_device(F[k * h:].data_ptr(), U[k * h:].data_ptr(), h, cfg)
for k in range(2):
    run(k, 3)
torch.cuda.synchronize()
t = time.perf_counter()
th = [threading.Thread(target=run, args=(k, 10)) for k in range(2)]
for x in th: x.start()
for x in th: x.join()
torch.cuda.synchronize()
t2 = (time.perf_counter() - t) / 10
print(f"two contexts x {h} sources, concurrent: {t2 * 1e3:.2f} ms per step (x{t1 / t2:.2f})", flush=True)
