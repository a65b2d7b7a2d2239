"""Pins of the oracle's Chebyshev inner inverses (reading R22; CPU).

* the recurrence reproduces the closed-form Chebyshev residual polynomial
  p_m(lam) = T_m((theta - lam) / delta) / T_m(theta / delta) on a diagonal operator;
* with the exact spectrum and many steps it reaches the direct solve;
* the Gershgorin bound bounds the spectrum of D^{-1} M;
* the outer iteration keeps the backward-Euler fixed point for P~1 and P~2;
* on config 1 two Chebyshev steps reduce the residual faster per outer iteration (recorded).
"""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from numpy.polynomial import chebyshev as C

import oracle
from oracle import chebyshev as ch
from oracle import extras
from workloads import make_problem, config_problem, load_scales, initial_iterate


@pytest.mark.parametrize("m", [1, 2, 5, 9])
def test_closed_form_polynomial(m):
    rng = np.random.default_rng(1)
    lam = rng.uniform(0.3, 4.0, 40)
    b = rng.standard_normal(40)
    lmin, lmax = 0.2, 4.5
    y = ch.chebyshev(sp.diags(lam).tocsr(), np.ones(40), b, m, lmin, lmax)
    theta, delta = (lmax + lmin) / 2, (lmax - lmin) / 2
    Tm = C.Chebyshev.basis(m)
    p = Tm((theta - lam) / delta) / Tm(theta / delta)
    assert np.allclose(y, (1.0 - p) / lam * b, rtol=1e-12, atol=1e-14)


def _blocks():
    prob = make_problem(2, 4, 2, 0.1, 1, storage=1e-3, kappa_median=1e-2, kappa_sigma=1.0, kappa_seed=2)
    S = oracle.OracleSystem(prob)
    P = ch.ChebyshevPrecond(S, 1)
    return S, P


def test_gershgorin_bounds_and_direct_limit():
    S, P = _blocks()
    for M, Dinv, lmax in ((P.A, S.DAinv, P.lmax_u), (P.St, S.DSinv, P.lmax_p)):
        f = Dinv != 0
        Mf = M[f][:, f].toarray()
        dh = np.sqrt(Dinv[f])
        ev = np.linalg.eigvalsh(dh[:, None] * Mf * dh[None, :])
        assert ev.max() <= lmax * (1 + 1e-12) and ev.min() > 0
        b = np.random.default_rng(3).standard_normal(f.sum())
        y = ch.chebyshev(sp.csr_matrix(Mf), Dinv[f], b, 400, ev.min(), ev.max())
        assert np.abs(y - np.linalg.solve(Mf, b)).max() < 1e-10 * np.abs(np.linalg.solve(Mf, b)).max()


@pytest.mark.parametrize("precond", [1, 2])
def test_fixed_point_is_backward_euler(precond):
    prob = make_problem(2, 3, 6, 1.0 / 6, 1, storage=1e-3, kappa_median=1e-2)
    S = oracle.OracleSystem(prob)
    s = load_scales(6, parity=True)
    X = np.zeros((7, S.ndof))
    X[1:] = S.to_paper(initial_iterate(prob.dirichlet, np.arange(1, 7), 5))
    X, h = ch.iterate(S, X, s, 2500, 4, precond, 0.5 if precond == 2 else 0.3)
    Xbe = extras.sequential_be(S, np.zeros(S.ndof), s, 6)
    assert np.abs(X - Xbe).max() / np.abs(Xbe).max() < 1e-11


def test_two_steps_converge_faster_config1():
    """Recorded behaviour (R22): with omega = 0.5 two Chebyshev steps reduce the
    total residual of config 1 by 0.23 in 100 outer iterations against 0.33 for the
    (scaled) diagonal inverse; more steps approach the exact inner inverse, with which
    the damped Richardson outer iteration itself needs a smaller omega."""
    prob = config_problem(1)
    S = oracle.OracleSystem(prob)
    nt = prob.n_t
    s = np.ones(nt)
    X = np.zeros((nt + 1, S.ndof))
    tot = {}
    for m in (1, 2):
        _, h = ch.iterate(S, X, s, 100, m, 2, 0.5)
        t = np.sqrt((h ** 2).sum(axis=(1, 2)))
        assert np.all(np.diff(t) <= 0)
        tot[m] = t[-1] / t[0]
    assert tot[2] < 0.8 * tot[1], tot
