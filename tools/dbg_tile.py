import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import oracle
from paper_2310_10430_b200 import BiotSolver
from workloads import config_problem, initial_iterate, load_scales
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prob = config_problem(cid)
nt = prob.n_t
s = load_scales(nt, parity=True)
W = 14
x0 = initial_iterate(prob.dirichlet, np.arange(1, W + 1), prob.x0_seed)
S = oracle.OracleSystem(prob)
X = np.zeros((W + 1, S.ndof)); X[1:] = S.to_paper(x0)
X, _ = S.iterate(X, s[:W], K, 2, 0.5, history=False)
xo = S.from_paper(X[1:])
for rep in range(2):
    for k in ("generic", "tile"):
        os.environ["BIOT_KERNEL"] = k
        g = BiotSolver(prob, precond=2, omega=0.5, load_scale=s)
        g.set_iterate(1, x0)
        g.iterate(K)
        xg = g.solution(1, W)
        d = np.abs(xg - xo).reshape(W, -1, prob.dim + 1).max(axis=(0, 2))
        bad = np.nonzero(d > 1e-9 * np.abs(xo).max())[0]
        print(rep, k, "path", g.info.kernel_path, "max err", d.max(), "bad", bad.size, bad[:10], flush=True)
        g.close()
