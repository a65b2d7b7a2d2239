"""Pins of the oracle's per-step GMRES (Alg. 3; CPU).

* one GMRES(k) cycle equals the definition: the minimiser of ||P^{-1}(b - AA x)|| over
  x0 + K_k(P^{-1} AA, P^{-1} r0), computed here from an explicit Krylov matrix;
* with k = the system size it is the direct solve;
* Alg. 3 with Gauss-Seidel in time and exact per-step solves is backward Euler after ONE
  outer iteration ("exactly consistent ... when N_thread = 1");
* the preconditioned residual never grows within a cycle; the outer iteration converges
  to the backward-Euler fixed point with Jacobi in time.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle
from oracle import extras
from oracle import gmres as gm
from workloads import make_problem, load_scales, initial_iterate


def _sys(n=3, nt=4):
    prob = make_problem(2, n, nt, 1.0 / nt, 1, storage=1e-3, kappa_median=1e-2, kappa_sigma=1.0, kappa_seed=4)
    return prob, oracle.OracleSystem(prob)


def test_cycle_is_the_krylov_minimiser():
    prob, S = _sys()
    rng = np.random.default_rng(2)
    f = S.free > 0
    x = rng.standard_normal(S.ndof) * S.free
    b = rng.standard_normal(S.ndof) * S.free
    for k in (1, 2, 3, 4):
        xn, beta, rn = gm.gmres_cycle(S, x, b, k)
        r0 = gm.apply_p2inv(S, b - S.AA @ x)
        Kcols = [r0]
        for _ in range(k - 1):
            Kcols.append(gm.apply_p2inv(S, S.AA @ Kcols[-1]))
        Km = np.column_stack(Kcols)
        MK = np.column_stack([gm.apply_p2inv(S, S.AA @ Km[:, j]) for j in range(k)])
        c = np.linalg.lstsq(MK[f], r0[f], rcond=None)[0]
        xk = x + Km @ c
        assert np.abs(xn - xk).max() <= 1e-7 * np.abs(xk - x).max()
        assert rn <= beta * (1 + 1e-12)


def test_full_dimension_is_direct_solve():
    prob, S = _sys(n=2)
    f = S.free > 0
    rng = np.random.default_rng(5)
    b = rng.standard_normal(S.ndof) * S.free
    xn, _, rn = gm.gmres_cycle(S, np.zeros(S.ndof), b, int(f.sum()))
    AAf = S.AA[f][:, f].tocsc()
    xd = spla.spsolve(AAf, b[f])
    assert np.abs(xn[f] - xd).max() < 1e-9 * np.abs(xd).max()


def test_gauss_seidel_exact_solves_are_backward_euler_in_one_iteration():
    prob, S = _sys(n=2, nt=5)
    s = load_scales(5, parity=True)
    X = np.zeros((6, S.ndof))
    X, _ = gm.iterate(S, X, s, 1, int((S.free > 0).sum()), gauss_seidel=True)
    Xbe = extras.sequential_be(S, np.zeros(S.ndof), s, 5)
    assert np.abs(X - Xbe).max() < 1e-9 * np.abs(Xbe).max()


def test_jacobi_outer_iteration_converges_to_backward_euler():
    prob, S = _sys(n=3, nt=4)
    s = load_scales(4, parity=True)
    X = np.zeros((5, S.ndof))
    X[1:] = S.to_paper(initial_iterate(prob.dirichlet, np.arange(1, 5), 7))
    X, h = gm.iterate(S, X, s, 40, 8)
    Xbe = extras.sequential_be(S, np.zeros(S.ndof), s, 4)
    assert np.abs(X - Xbe).max() < 1e-9 * np.abs(Xbe).max()
