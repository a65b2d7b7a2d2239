"""Dev aid: tile3d vs generic kernel on a small 3D case; prints where they differ."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_10430_b200 import BiotSolver
from workloads import make_problem, initial_iterate, load_scales

n, nt, S, sig = [float(v) for v in sys.argv[1:5]] if len(sys.argv) > 4 else (7, 40, 1e-3, 1.0)
n, nt = int(n), int(nt)
K = int(sys.argv[5]) if len(sys.argv) > 5 else 1
prob = make_problem(3, n, nt, 0.01, 6, storage=S, kappa_median=1e-3, kappa_sigma=sig, kappa_seed=3, x0_seed=9)
res = {}
for kern in ("generic", "tile"):
    os.environ["BIOT_KERNEL"] = kern
    s = load_scales(nt, parity=True)
    g = BiotSolver(prob, n_t=nt, load_scale=s, precond=2)
    g.set_iterate(1, initial_iterate(prob.dirichlet, np.arange(1, nt + 1), prob.x0_seed))
    g.iterate(K)
    res[kern] = (g.solution(), g.residual_history(K - 1), g.info.kernel_path)
    g.close()
x, ref = res["tile"][0], res["generic"][0]
n1 = n + 1
d = np.abs(x - ref).reshape(nt, n1, n1, n1, 4)
print("paths", res["generic"][2], res["tile"][2], "max rel", d.max() / np.abs(ref).max())
bad = np.argwhere(d > 1e-12 * np.abs(ref).max())
print("n bad", len(bad))
for b in bad[:20]:
    print("t,z,y,x,c", b, d[tuple(b)])
h, hr = res["tile"][1], res["generic"][1]
print("hist rel", np.abs(h - hr).max() / np.abs(hr).max())
