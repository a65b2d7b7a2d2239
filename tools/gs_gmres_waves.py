"""Run the first W waves of a Gauss-Seidel + GMRES(k) run with K sweeps in flight on a
config (for an ncu launch list of the steady-state waves).  Dev tool.

    python tools/gs_gmres_waves.py [config] [K] [k] [waves]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2310_10430_b200 import BiotSolver  # noqa: E402
from workloads import config_problem  # noqa: E402

cid, K, k, W = (int(a) for a in (sys.argv[1:] + ["3", "16", "10", "64"][len(sys.argv) - 1:]))
g = BiotSolver(config_problem(cid), precond=2, omega=1.0)
g.gs_begin(K, k)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(W):
    g.gs_wave()
torch.cuda.synchronize()
print(f"config {cid}: {W} waves of GS + GMRES({k}), K = {K}: {(time.perf_counter() - t0) / W * 1e3:.2f} ms per wave")
g.close()
