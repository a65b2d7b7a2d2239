"""Small runs of every tile-kernel mode for compute-sanitizer (racecheck / synccheck /
memcheck): tile2d and tile3d, P~2 and P~1, multi-chunk and single-chunk passes, the
residual-only pass, Gauss-Seidel windows, GMRES (ZOUT / MATVEC).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2310_10430_b200 import BiotSolver  # noqa: E402
from workloads import config_problem, make_problem, initial_iterate, load_scales  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def run(prob, nt, precond, tag, gs=False, gmres=0):
    s = load_scales(nt, parity=True)
    g = BiotSolver(prob, n_t=nt, precond=precond, omega=0.5 if precond == 2 else 0.3, load_scale=s)
    g.set_iterate(1, initial_iterate(prob.dirichlet, np.arange(1, nt + 1), 5))
    if gs:
        g.iterate_gs(2)
    elif gmres:
        g.iterate_gmres(1, gmres)
    else:
        g.iterate(2)
    r = g.residual_norms()
    info = g.get_info()
    g.close()
    print(f"{tag}: kernel_path={info.kernel_path} ok, |r|={np.sqrt((r ** 2).sum()):.3e}", flush=True)


p2 = config_problem(1)
p3 = make_problem(3, 9, 40, 0.01, 2, storage=1e-3, kappa_median=1e-3, kappa_sigma=1.0, kappa_seed=3)
if which in ("all", "2d"):
    for pc in (2, 1):
        run(p2, 200, pc, f"tile2d P~{pc} N_t=200 (2 chunks, ragged)")
        run(p2, 32, pc, f"tile2d P~{pc} N_t=32 (single chunk)")
        run(p2, 40, pc, f"tile2d P~{pc} Gauss-Seidel windows", gs=True)
    run(p2, 32, 2, "tile2d GMRES(3)", gmres=3)
if which in ("all", "3d"):
    for pc in (2, 1):
        run(p3, 40, pc, f"tile3d P~{pc} N_t=40 (2 chunks, ragged)")
        run(p3, 12, pc, f"tile3d P~{pc} Gauss-Seidel windows", gs=True)
    run(p3, 20, 2, "tile3d GMRES(3)", gmres=3)
print("sanitize_run done")
