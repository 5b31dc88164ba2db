"""Wall-clock split of the offline stage on the GPU (PT_OFFLINE_TIMES): python tools/offline_times.py cfg5 [k1|torch]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PT_OFFLINE_TIMES"] = "1"
import torch

from paper_1510_01831_b200.configs import make_config
from paper_1510_01831_b200.offline import build_factors

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
route = sys.argv[2] if len(sys.argv) > 2 else "k1"
prob = make_config(name)
torch.cuda.synchronize()
t = time.perf_counter()
F = build_factors(prob.grid, prob.model, prob.pml, prob.partition, prob.Lc, device="cuda", cell_solver=route)
torch.cuda.synchronize()
print(f"{name} offline ({route}): {time.perf_counter() - t:.2f}s, peak HBM {torch.cuda.max_memory_allocated() / 1e9:.1f} GB")
