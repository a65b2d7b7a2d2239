"""Pins of the oracle's iteration (CPU only, no GPU).

* fixed point == sequential backward Euler by direct solve;
* first iterate closed form and the preconditioner inverse relation P^ z = r;
* Jacobi-in-time light cone / window / front invariants (bitwise);
* monotone residual within K at configs 1-2 (BJ: "residual must decrease");
* Terzaghi closed form under (h, tau) refinement (physics);
* negative control: the undamped literal iteration diverges (R1/R3).
"""
import numpy as np
import pytest

import oracle
from oracle import extras
from workloads import make_problem, config_problem, load_scales, initial_iterate


def _rand_run(prob, S, nt, seed=5):
    x0 = initial_iterate(prob.dirichlet, np.arange(1, nt + 1), seed)
    X = np.zeros((nt + 1, S.ndof))
    X[1:] = S.to_paper(x0)
    return X


@pytest.mark.parametrize("dim,n,nt,K,omega", [(2, 2, 4, 3000, 0.5), (2, 4, 8, 8000, 0.5),
                                               (3, 1, 4, 3000, 0.5), (3, 2, 4, 6000, 0.5)])
@pytest.mark.parametrize("precond", [1, 2])
def test_fixed_point_is_backward_euler(dim, n, nt, K, omega, precond):
    prob = make_problem(dim, n, nt, 1.0 / nt, K, storage=1e-3, kappa_median=1e-2)
    S = oracle.OracleSystem(prob)
    s = load_scales(nt, parity=True)
    X = _rand_run(prob, S, nt)
    X, hist = S.iterate(X, s, K, precond, omega, history=False)
    Xbe = extras.sequential_be(S, np.zeros(S.ndof), s, nt)
    err = np.abs(X - Xbe).max() / np.abs(Xbe).max()
    assert err < 1e-11, err
    assert S.residual_norms(X, s).max() < 1e-11 * np.abs(S.F).max() + 1e-13


@pytest.mark.parametrize("precond", [1, 2])
@pytest.mark.parametrize("omega", [0.5, 0.3])
def test_first_iterate_and_preconditioner_inverse(precond, omega):
    """x^0 = 0: x_n^1 = omega P^-1 s_n f, checked as P^ (x_n^1/omega) = s_n f with
    P^ = [[diag A, 0], [B^T (P~1 only), -diag S~p]] built from the blocks."""
    prob = make_problem(2, 6, 5, 0.2, 1)
    S = oracle.OracleSystem(prob)
    s = load_scales(5, parity=True)
    X = np.zeros((6, S.ndof))
    X, _ = S.iterate(X, s, 1, precond, omega)
    free = S.free > 0
    fu, fp = free[:S.nu], free[S.nu:]
    Dd = np.concatenate([S.blocks.A.diagonal(), -S.St.diagonal()])
    for n in range(1, 6):
        z = X[n] / omega
        Pz = Dd * z
        if precond == 1:
            Pz[S.nu:] += S.blocks.B.T @ (z[:S.nu] * fu)
        rhs = s[n - 1] * S.F
        assert np.allclose(Pz[free], rhs[free], rtol=1e-13, atol=1e-16)
        assert np.all(z[~free] == 0)
    if precond == 2:
        assert np.abs(X[1:, S.nu:]).max() == 0.0    # f_p = 0 and block-diagonal P


def test_jacobi_light_cone_window_front():
    prob = config_problem(1)
    S = oracle.OracleSystem(prob)
    nt, K = prob.n_t, 6
    s = load_scales(nt, parity=True)
    X0 = _rand_run(prob, S, nt)
    Xf, _ = S.iterate(X0.copy(), s, K, 2, 0.5, history=False)
    # truncation: steps <= M do not see steps > M
    M = 13
    Xt, _ = S.iterate(X0[:M + 1].copy(), s[:M], K, 2, 0.5, history=False)
    assert np.array_equal(Xt, Xf[:M + 1])
    # window [ns, nt] with an arbitrary ghost is exact for n >= ns + K
    ns = 10
    Xw = X0[ns - 1:].copy()
    Xw[0] = np.random.default_rng(9).standard_normal(S.ndof) * S.free
    Xw, _ = S.iterate(Xw, s[ns - 1:], K, 2, 0.5, history=False)
    assert np.array_equal(Xw[K + 1:], Xf[ns + K:])
    assert not np.array_equal(Xw[1], Xf[ns])               # the ghost does matter inside the cone
    # front: x^0 = 0, s = 1 -> x_n^K = x_K^K for n >= K
    Xz, _ = S.iterate(np.zeros_like(X0), np.ones(nt), K, 1, 0.5, history=False)
    for n in range(K, nt + 1):
        assert np.array_equal(Xz[n], Xz[K])
    assert not np.array_equal(Xz[K - 1], Xz[K])
    # Gauss-Seidel-in-time (Alg. 2 literal) differs after one sweep but shares the fixed point
    Xg = extras.gauss_seidel_in_time(S, X0, s, 1)
    Xj, _ = S.iterate(X0.copy(), s, 1, 2, 0.5, history=False)
    assert np.array_equal(Xg[1], Xj[1]) and not np.allclose(Xg[2:], Xj[2:])


@pytest.mark.parametrize("cid", [1, 2])
@pytest.mark.parametrize("precond", [1, 2])
def test_monotone_residual_metric_inputs(cid, precond):
    prob = config_problem(cid)
    S = oracle.OracleSystem(prob)
    nt, K = prob.n_t, prob.K
    if cid == 2:
        K = 25      # CPU time; full K=100 is covered in the GPU history test
    X = np.zeros((nt + 1, S.ndof))
    X, h = S.iterate(X, np.ones(nt), K, precond, 0.5)
    tot = np.sqrt((h ** 2).sum(axis=(1, 2)))
    assert np.all(np.diff(tot) <= 0), tot
    assert tot[-1] < tot[0]
    fin = S.residual_norms(X, np.ones(nt))
    assert np.sqrt((fin ** 2).sum()) <= tot[-1]
    # norms at x = 0 are s_n ||f_u|| and 0 (x_0 = 0)
    assert np.allclose(h[0, :, 0], np.linalg.norm(S.F[:S.nu]), rtol=1e-14)
    assert np.abs(h[0, :, 1]).max() == 0.0


def test_negative_control_undamped_diverges():
    """Exact P~1/P~2 with omega=1 (the literal Alg. 1-2 update) diverge at config 1;
    the diagonal P^ damped by omega=0.5 contracts (readings R1-R3)."""
    S = oracle.OracleSystem(config_problem(1))
    assert extras.spectral_radius(extras.iteration_matrix(S, 1, True, 1.0)) > 10
    assert extras.spectral_radius(extras.iteration_matrix(S, 2, True, 1.0)) > 2
    for pc in (1, 2):
        assert extras.spectral_radius(extras.iteration_matrix(S, pc, False, 1.0)) > 1
        assert extras.spectral_radius(extras.iteration_matrix(S, pc, False, 0.5)) < 1


def _terzaghi_err(n, nt, storage):
    prob = make_problem(2, n, nt, 1.0 / nt, 1, lam=1.0, mu=1.0, alpha=1.0, storage=storage,
                        kappa_median=1e-2)
    # drained top with kappa=1e-2 is slow; use kappa=1 and t=1/... scaled: keep config-1 physics
    S = oracle.OracleSystem(prob)
    X = extras.sequential_be(S, np.zeros(S.ndof), np.ones(nt), nt)
    x = S.from_paper(X[nt]).reshape(-1, 3)
    y = prob.coords[:, 1]
    pex = extras.terzaghi_p(y, 1.0, 1.0, 1.0, 1.0, storage, 1e-2)
    uex = extras.terzaghi_uy(y, 1.0, 1.0, 1.0, 1.0, storage, 1e-2)
    return np.abs(x[:, 2] - pex).max(), np.abs(x[:, 1] - uex).max()


@pytest.mark.parametrize("storage", [1e-3, 0.5])
def test_terzaghi_column(storage):
    """Converged BE of the config-1 column vs the 1-D consolidation series at t=1."""
    e16, u16 = _terzaghi_err(16, 32, storage)
    e32, u32 = _terzaghi_err(32, 64, storage)
    e64, u64 = _terzaghi_err(64, 128, storage)
    assert e16 < 0.07 and e32 < 0.04 and e64 < 0.022, (e16, e32, e64)
    assert e16 / e32 > 1.5 and e32 / e64 > 1.6          # first order in (h, tau)
    assert u64 < u16 and u64 < 0.01


# ---- Gauss-Seidel in time (Algorithm 2 read literally) ----

@pytest.mark.parametrize("dim,n,nt,K", [(2, 3, 6, 4000), (3, 1, 4, 3000)])
@pytest.mark.parametrize("precond", [1, 2])
def test_gs_fixed_point_is_backward_euler(dim, n, nt, K, precond):
    """GS-in-time converges to the same sequential BE solution (direct solve)."""
    prob = make_problem(dim, n, nt, 1.0 / nt, K, storage=1e-3, kappa_median=1e-2)
    S = oracle.OracleSystem(prob)
    s = load_scales(nt, parity=True)
    X = extras.gauss_seidel_in_time(S, _rand_run(prob, S, nt), s, K, precond, 0.5)
    Xbe = extras.sequential_be(S, np.zeros(S.ndof), s, nt)
    assert np.abs(X - Xbe).max() / np.abs(Xbe).max() < 1e-11


def test_gs_single_step_equals_jacobi_and_step_one_is_sequential():
    """N_t = 1: GS and Jacobi are the same iteration (bitwise); step 1 of GS never sees a
    changing predecessor, so after m sweeps it equals m Jacobi sweeps of step 1 alone."""
    prob = make_problem(2, 4, 1, 0.1, 7, storage=1e-3, kappa_median=1e-2)
    S = oracle.OracleSystem(prob)
    s = load_scales(1, parity=True)
    X0 = _rand_run(prob, S, 1)
    for pc in (1, 2):
        Xg, hg = extras.gauss_seidel_in_time(S, X0, s, 7, pc, 0.5, history=True)
        Xj, hj = S.iterate(X0.copy(), s, 7, pc, 0.5)
        assert np.array_equal(Xg, Xj)
        assert np.allclose(hg, hj, rtol=1e-13, atol=0)
    prob4 = make_problem(2, 4, 5, 0.1, 6, storage=1e-3, kappa_median=1e-2)
    S4 = oracle.OracleSystem(prob4)
    s4 = load_scales(5, parity=True)
    X4 = _rand_run(prob4, S4, 5)
    Xg = extras.gauss_seidel_in_time(S4, X4, s4, 6)
    Xj, _ = S4.iterate(X4[:2].copy(), s4[:1], 6, 2, 0.5, history=False)
    assert np.array_equal(Xg[1], Xj[1])


def test_gs_causality_one_sweep_reaches_every_step():
    """With no load (s = 0) and x^0 = 0 except step 1, one GS sweep carries the
    perturbation to every later step (b^{n,m} uses X^{n-1,m}), one Jacobi sweep
    only to step 2 (the information fronts of the two schemes)."""
    prob = make_problem(2, 3, 6, 0.1, 1, storage=1e-3, kappa_median=1e-2)
    S = oracle.OracleSystem(prob)
    s = np.zeros(6)
    X = np.zeros((7, S.ndof))
    X[1] = S.to_paper(initial_iterate(prob.dirichlet, np.array([1]), 3))[0]
    Xg = extras.gauss_seidel_in_time(S, X, s, 1)
    Xj, _ = S.iterate(X.copy(), s, 1, 2, 0.5, history=False)
    assert all(np.abs(Xg[n]).max() > 0 for n in range(1, 7))
    assert np.abs(Xj[2]).max() > 0 and all(np.abs(Xj[n]).max() == 0 for n in range(3, 7))

