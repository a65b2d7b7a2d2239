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


def _dense_phat(S, precond):
    """The preconditioner matrix itself on the free DoFs, built from the blocks (not from
    apply_*inv): P^1 = [[D_A, 0], [B^T, -D_S]], P^2 = [[D_A, 0], [0, -D_S]] (eqs. p1/p2, R2)."""
    nu = S.nu
    DA = np.where(S.DAinv != 0, 1.0 / np.where(S.DAinv != 0, S.DAinv, 1.0), 0.0)
    DS = np.where(S.DSinv != 0, 1.0 / np.where(S.DSinv != 0, S.DSinv, 1.0), 0.0)
    P = np.zeros((S.ndof, S.ndof))
    P[np.arange(nu), np.arange(nu)] = DA
    P[nu + np.arange(S.np), nu + np.arange(S.np)] = -DS
    if precond == 1:
        P[nu:, :nu] = (S.blocks.B.T.toarray() * S.free[nu:, None]) * S.free[None, :nu]
    return P


@pytest.mark.parametrize("precond", [2, 1])
def test_preconditioner_apply_inverts_the_block_matrix(precond):
    """apply_pinv(r) solves P^ z = r on the free DoFs (the lower-triangular P~1 block
    structure with its sign, eq. p1: a dropped B^T term or a flipped sign fails)."""
    prob, S = _sys()
    f = S.free > 0
    rng = np.random.default_rng(9)
    r = rng.standard_normal(S.ndof) * S.free
    z = gm.apply_pinv(S, r, precond)
    P = _dense_phat(S, precond)
    assert np.abs((P @ z - r)[f]).max() < 1e-12 * np.abs(r).max()
    assert np.abs(z[~f]).max() == 0.0


@pytest.mark.parametrize("precond", [2, 1])
def test_cycle_is_the_krylov_minimiser(precond):
    prob, S = _sys()
    rng = np.random.default_rng(2)
    f = S.free > 0
    x = rng.standard_normal(S.ndof) * S.free
    b = rng.standard_normal(S.ndof) * S.free
    for k in (1, 2, 3, 4):
        xn, beta, rn = gm.gmres_cycle(S, x, b, k, precond)
        r0 = gm.apply_pinv(S, b - S.AA @ x, precond)
        Kcols = [r0]
        for _ in range(k - 1):
            Kcols.append(gm.apply_pinv(S, S.AA @ Kcols[-1], precond))
        Km = np.column_stack(Kcols)
        MK = np.column_stack([gm.apply_pinv(S, S.AA @ Km[:, j], precond) for j in range(k)])
        c = np.linalg.lstsq(MK[f], r0[f], rcond=None)[0]
        xk = x + Km @ c
        assert np.abs(xn - xk).max() <= 1e-7 * np.abs(xk - x).max()
        assert rn <= beta * (1 + 1e-12)


@pytest.mark.parametrize("precond", [2, 1])
def test_full_dimension_is_direct_solve(precond):
    prob, S = _sys(n=2)
    f = S.free > 0
    rng = np.random.default_rng(5)
    b = rng.standard_normal(S.ndof) * S.free
    xn, _, rn = gm.gmres_cycle(S, np.zeros(S.ndof), b, int(f.sum()), precond)
    AAf = S.AA[f][:, f].tocsc()
    xd = spla.spsolve(AAf, b[f])
    assert np.abs(xn[f] - xd).max() < 1e-9 * np.abs(xd).max()


@pytest.mark.parametrize("precond", [2, 1])
def test_gauss_seidel_exact_solves_are_backward_euler_in_one_iteration(precond):
    prob, S = _sys(n=2, nt=5)
    s = load_scales(5, parity=True)
    X = np.zeros((6, S.ndof))
    X, _ = gm.iterate(S, X, s, 1, int((S.free > 0).sum()), gauss_seidel=True, precond=precond)
    Xbe = extras.sequential_be(S, np.zeros(S.ndof), s, 5)
    assert np.abs(X - Xbe).max() < 1e-9 * np.abs(Xbe).max()


@pytest.mark.parametrize("precond", [2, 1])
def test_jacobi_outer_iteration_converges_to_backward_euler(precond):
    prob, S = _sys(n=3, nt=4)
    s = load_scales(4, parity=True)
    X = np.zeros((5, S.ndof))
    X[1:] = S.to_paper(initial_iterate(prob.dirichlet, np.arange(1, 5), 7))
    X, h = gm.iterate(S, X, s, 40, 8, precond=precond)
    Xbe = extras.sequential_be(S, np.zeros(S.ndof), s, 4)
    assert np.abs(X - Xbe).max() < 1e-9 * np.abs(Xbe).max()
