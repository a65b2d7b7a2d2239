import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_2310_10430_b200 import BiotSolver, FLAG_MANUAL_HALO, FLAG_DEFER_STEP0
from workloads import trig_problem, initial_iterate, load_scales
tp = trig_problem(4, 64, 1.0 / 64)
nt, world, K = 64, 4, int(sys.argv[1]) if len(sys.argv) > 1 else 1
for pc in (2, 1):
    s = load_scales(nt, parity=True)
    def seeded(**kw):
        g = BiotSolver(tp, n_t=nt, load_scale=s, precond=pc, omega=0.5 if pc == 2 else 0.3, **kw)
        g.set_iterate(g.first_step, initial_iterate(tp.dirichlet, np.arange(g.first_step, g.first_step + g.n_tl), tp.x0_seed))
        return g
    ref = seeded(); ref.iterate(K); xr = ref.solution()
    for flags in (FLAG_MANUAL_HALO, FLAG_MANUAL_HALO | FLAG_DEFER_STEP0):
        ranks = [seeded(rank=r, world=world, flags=flags) for r in range(world)]
        for _ in range(K):
            sl = [g.last_slice() for g in ranks]
            for r in range(1, world): ranks[r].set_ghost(sl[r - 1])
            for g in ranks: g.iterate(1)
        xs = np.concatenate([g.solution() for g in ranks]).reshape(nt, -1, 3)
        d = np.abs(xs - xr.reshape(nt, -1, 3))
        bad = np.argwhere(d > 0)
        print("P~%d flags %d maxdiff %.3e nbad %d steps %s comps %s" % (pc, flags, d.max(), len(bad), np.unique(bad[:, 0])[:20], np.unique(bad[:, 2])))
