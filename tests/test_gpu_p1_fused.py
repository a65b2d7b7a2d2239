"""Single-pass P~1 (tile2d MODE_P1_FUSED, PAPER.md eq. p1) against the two-pass form
(BIOT_P1_TWOPASS=1: residual pass writing the Z panel, then z_p = D_S^{-1}(B^T z_u - r_p))
and against the oracle.  Both compute the same B^T z_u in the same slot order; they differ
only in how x_p + omega D_S^{-1}(bt - r_p) is rounded, so they agree to ~1e-15 relative.
"""
import os

import numpy as np
import pytest

import oracle
from paper_2310_10430_b200 import BiotSolver
from workloads import config_problem, make_problem, initial_iterate, load_scales, trig_problem

from _parity import TOL, field_errors, norm_errors

pytestmark = pytest.mark.gpu


def _solver(prob, nt, twopass, **kw):
    old = os.environ.get("BIOT_P1_TWOPASS")
    os.environ["BIOT_P1_TWOPASS"] = "1" if twopass else "0"
    try:
        return BiotSolver(prob, n_t=nt, precond=1, **kw)
    finally:
        if old is None:
            del os.environ["BIOT_P1_TWOPASS"]
        else:
            os.environ["BIOT_P1_TWOPASS"] = old


def _run(prob, nt, K, twopass, gs=False, omega=0.3):
    s = load_scales(nt, parity=True)
    g = _solver(prob, nt, twopass, omega=omega, load_scale=s)
    try:
        g.set_iterate(1, initial_iterate(prob.dirichlet, np.arange(1, nt + 1), prob.x0_seed))
        (g.iterate_gs if gs else g.iterate)(K)
        info = g.get_info()
        return g.solution(), np.stack([g.residual_history(k) for k in range(K)]), g.residual_norms(), info
    finally:
        g.close()


@pytest.mark.parametrize("cid,nt,K", [(1, 32, 20), (2, 256, 7), (2, 300, 3)])
def test_fused_matches_two_pass_and_oracle(cid, nt, K):
    prob = config_problem(cid)
    xf, hf, rf, inf_f = _run(prob, nt, K, False)
    xt, ht, rt, inf_t = _run(prob, nt, K, True)
    assert inf_f.launches_per_iter < inf_t.launches_per_iter     # one pass instead of two
    assert field_errors(xf, xt, 2).max() < 1e-13
    assert norm_errors(hf.reshape(-1, 2), ht.reshape(-1, 2)).max() < 1e-13
    s = load_scales(nt, parity=True)
    x0 = initial_iterate(prob.dirichlet, np.arange(1, nt + 1), prob.x0_seed)
    xo, ho, S = oracle.run(prob, x0, s, K, 1, 0.3)
    assert field_errors(xf, xo, 2).max() < TOL
    assert norm_errors(hf.reshape(-1, 2), ho.reshape(-1, 2)).max() < TOL
    ro = S.residual_norms(np.vstack([np.zeros(S.ndof), S.to_paper(xo)]), s)
    assert norm_errors(rf, ro).max() < TOL


@pytest.mark.parametrize("n", [3, 9, 10, 11, 21, 23])
def test_fused_odd_widths(n):
    """Grid widths around the 10-column tile (one tile, exact multiples, a 1-column last
    tile) and rows per tile from 1 up: every halo/edge case of the fused tile."""
    prob = make_problem(2, n, 40, 0.01, 5, storage=1e-3, kappa_median=1e-2, kappa_sigma=1.0,
                        kappa_seed=5, x0_seed=3)
    for rows in ("1", "2", "5", ""):
        if rows:
            os.environ["BIOT_P1_ROWS"] = rows
        try:
            xf, hf, _, _ = _run(prob, 40, 5, False)
        finally:
            os.environ.pop("BIOT_P1_ROWS", None)
        xt, ht, _, _ = _run(prob, 40, 5, True)
        assert field_errors(xf, xt, 2).max() < 1e-13, (n, rows)
        assert norm_errors(hf.reshape(-1, 2), ht.reshape(-1, 2)).max() < 1e-13, (n, rows)


def test_fused_gauss_seidel_windows():
    prob = config_problem(1)
    xf, hf, _, _ = _run(prob, 40, 9, False, gs=True)
    xt, ht, _, _ = _run(prob, 40, 9, True, gs=True)
    assert field_errors(xf, xt, 2).max() < 1e-13
    assert norm_errors(hf.reshape(-1, 2), ht.reshape(-1, 2)).max() < 1e-13


def test_fused_trig_multiload():
    """§4.1 (four load terms: the kMaxLoads variant of the fused kernel)."""
    tp = trig_problem(5, 300, 1.0 / 300)
    xf, hf, _, _ = _run(tp, 300, 4, False)
    xt, ht, _, _ = _run(tp, 300, 4, True)
    assert field_errors(xf, xt, 2).max() < 1e-13
    assert norm_errors(hf.reshape(-1, 2), ht.reshape(-1, 2)).max() < 1e-13
