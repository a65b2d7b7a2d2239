"""§4.1 trigonometric test on the GPU -- needs a B200.

Multi-term loads (sources with cos/sin coefficients, Dirichlet lifting at c_n and
c_{n-1}; reading R24) through every iteration of the library, against the oracle at
1e-9 per field (R17): Jacobi in time with P~2 / P~1 on the 2D tile kernel and the
generic kernel, Gauss-Seidel in time, per-step GMRES and Alg. 3 (GS + GMRES).  Then
two consistency checks with closed forms: the affine patch solution is reproduced
exactly, and the converged h = 1/16, tau = 1/1024 solution has the oracle's backward-
Euler L2 error (Table 1 row 1 within the golden band).
"""
import numpy as np
import pytest

import oracle
from oracle import extras
from oracle import gmres as ogm
from paper_2310_10430_b200 import BiotSolver
from workloads import trig_problem, linear_patch_problem, patch_exact, initial_iterate

from _parity import TOL, field_errors, norm_errors

pytestmark = pytest.mark.gpu


def _x0(prob, nt):
    return initial_iterate(prob.dirichlet, np.arange(1, nt + 1), 31)


def _oracle_start(prob, nt, x0):
    S = oracle.OracleSystem(prob)
    C = S.coefs(np.zeros(nt), 1, nt)
    X = np.zeros((nt + 1, S.ndof))
    X[0] = S.to_paper(prob.x_initial) * S.free
    X[1:] = S.to_paper(x0)
    return S, C, X


def _solver(prob, nt, precond, omega, monkeypatch=None, generic=False):
    if monkeypatch is not None:
        if generic:
            monkeypatch.setenv("BIOT_KERNEL", "generic")
        else:
            monkeypatch.delenv("BIOT_KERNEL", raising=False)
    return BiotSolver(prob, n_t=nt, precond=precond, omega=omega)


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("precond,omega", [(2, 0.5), (1, 0.3)])
@pytest.mark.parametrize("k,nt,K", [(4, 40, 20), (5, 300, 6)])
def test_trig_parity_jacobi(monkeypatch, generic, precond, omega, k, nt, K):
    prob = trig_problem(k, nt, 1.0 / 64)
    x0 = _x0(prob, nt)
    g = _solver(prob, nt, precond, omega, monkeypatch, generic)
    try:
        assert g.info.kernel_path == (1 if generic else 5)
        g.set_iterate(1, x0)
        g.iterate(K)
        xg = g.solution()
        hg = np.stack([g.residual_history(kk) for kk in range(K)])
        rg = g.residual_norms()
    finally:
        g.close()
    S, C, X = _oracle_start(prob, nt, x0)
    Xo, ho = S.iterate(X, C, K, precond, omega)
    ro = S.residual_norms(Xo, C)
    xo = np.stack([S.from_paper(v) for v in Xo[1:]])
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL
    assert norm_errors(rg, ro).max() < TOL


@pytest.mark.parametrize("precond,omega", [(2, 0.5), (1, 0.3)])
def test_trig_parity_gs(precond, omega):
    nt, K = 50, 7
    prob = trig_problem(4, nt, 1.0 / 64)
    x0 = _x0(prob, nt)
    g = BiotSolver(prob, n_t=nt, precond=precond, omega=omega)
    try:
        g.set_iterate(1, x0)
        g.iterate_gs(K)
        xg = g.solution()
        hg = np.stack([g.residual_history(kk) for kk in range(K)])
    finally:
        g.close()
    S, C, X = _oracle_start(prob, nt, x0)
    Xo, ho = extras.gauss_seidel_in_time(S, X, C, K, precond, omega, history=True)
    xo = np.stack([S.from_paper(v) for v in Xo[1:]])
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


@pytest.mark.parametrize("gs", [False, True])
def test_trig_parity_gmres(gs):
    nt, K, k = 33, 3, 5
    prob = trig_problem(4, nt, 1.0 / 64)
    x0 = _x0(prob, nt)
    g = BiotSolver(prob, n_t=nt, precond=2, omega=0.5)
    try:
        g.set_iterate(1, x0)
        (g.iterate_gs_gmres if gs else g.iterate_gmres)(K, k)
        xg = g.solution()
        hg = np.stack([g.residual_history(kk) for kk in range(K)])
    finally:
        g.close()
    S, C, X = _oracle_start(prob, nt, x0)
    Xo, ho = ogm.iterate(S, X, C, K, k, gauss_seidel=gs)
    xo = np.stack([S.from_paper(v) for v in Xo[1:]])
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


def test_patch_solution_exact_on_gpu():
    """The affine-in-space-and-time solution is a fixed point of the GPU iteration: from
    x^0 = 0 the Jacobi iteration converges to it (every load term enters)."""
    prob = linear_patch_problem(4, 8, 0.125)
    g = BiotSolver(prob, precond=2, omega=0.5)
    try:
        g.iterate(8000)
        x = g.solution()
    finally:
        g.close()
    fixed = np.asarray(prob.dirichlet, dtype=np.float64)
    for n in range(1, prob.n_t + 1):
        full = x[n - 1] + prob.dirichlet_coef[n] * prob.dirichlet_values * fixed
        ref = patch_exact(prob.coords, n * prob.dt)
        assert np.abs(full - ref).max() < 1e-9 * np.abs(ref).max()


def test_trig_converged_matches_backward_euler():
    """h = 1/16, tau = 1/1024, t = 1 (Table 1 row 1): Alg. 3 (GS + GMRES(16) per step)
    swept to convergence equals the oracle's sequential backward Euler, so its L2 error
    of p is the oracle's (pinned against Table 1 in test_oracle_trig)."""
    from test_oracle_trig import l2_error_p, full_field, be_solution
    nt = 1024
    prob = trig_problem(4, nt, 1.0 / 1024)
    S, C, Xbe = be_solution(prob)
    g = BiotSolver(prob, precond=2, omega=0.5)
    try:
        g.iterate_gs_gmres(1, 16)
        r0 = g.residual_norms().max()
        for sweep in range(60):
            g.iterate_gs_gmres(1, 16)
            if g.residual_norms().max() < 1e-11 * r0:
                break
        x = g.solution()
    finally:
        g.close()
    xbe = np.stack([S.from_paper(v) for v in Xbe[1:]])
    assert field_errors(x, xbe, 2).max() < 1e-8
    fixed = np.asarray(prob.dirichlet, dtype=np.float64)
    p = (x[nt - 1] + prob.dirichlet_coef[nt] * prob.dirichlet_values * fixed).reshape(-1, 3)[:, 2]
    pbe = full_field(prob, S, Xbe, nt).reshape(-1, 3)[:, 2]
    e, ebe = l2_error_p(prob, p, 1.0), l2_error_p(prob, pbe, 1.0)
    assert abs(e - ebe) < 1e-6 * ebe


@pytest.mark.parametrize("precond", [2, 1])
def test_trig_time_slabs_bitwise(precond):
    """Multi-load problem split into time slabs (manual halo): each slab takes the load
    coefficients of its global steps, the lifting of its first step uses c_{first-1}; the
    iterates equal the single-slab run bitwise."""
    from paper_2310_10430_b200 import FLAG_MANUAL_HALO
    nt, K, world = 256, 7, 2
    prob = trig_problem(5, nt, 1.0 / 256)
    x0 = _x0(prob, nt)
    omega = 0.5 if precond == 2 else 0.3
    ref = BiotSolver(prob, n_t=nt, precond=precond, omega=omega)
    ranks = [BiotSolver(prob, n_t=nt, precond=precond, omega=omega, rank=r, world=world, flags=FLAG_MANUAL_HALO)
             for r in range(world)]
    try:
        ref.set_iterate(1, x0)
        ref.iterate(K)
        for g in ranks:
            g.set_iterate(g.first_step, x0[g.first_step - 1:g.first_step - 1 + g.n_tl])
        for _ in range(K):
            sl = [g.last_slice() for g in ranks]
            for r in range(1, world):
                ranks[r].set_ghost(sl[r - 1])
            for g in ranks:
                g.iterate(1)
        xs = np.concatenate([g.solution() for g in ranks])
        assert np.array_equal(xs, ref.solution())
    finally:
        ref.close()
        for g in ranks:
            g.close()


@pytest.mark.parametrize("precond,omega", [(2, 0.5), (1, 0.3)])
def test_trig_parity_bench_size_windows(precond, omega):
    """The benchmark's §4.1 configuration (h = 1/512, N_t = 1024, the launch configuration
    bench.py --workload trig times): x^K on sampled step windows against the oracle run on a
    window that starts K steps earlier (light cone: x_n^K depends on x^0 of steps n-K..n
    only), with the load coefficients of the global steps."""
    nt, K = 1024, 4
    prob = trig_problem(9, nt, 1.0 / 1024)
    x0 = _x0(prob, nt)
    g = BiotSolver(prob, n_t=nt, precond=precond, omega=omega)
    try:
        g.set_iterate(1, x0)
        g.iterate(K)
        S = oracle.OracleSystem(prob)
        for n_lo, n_hi in [(1, 3), (517, 520), (1021, 1024)]:
            a = max(1, n_lo - K)
            L = n_hi - a + 1
            X = np.zeros((L + 1, S.ndof))
            X[0] = S.to_paper(x0[a - 2]) if a > 1 else S.to_paper(prob.x_initial) * S.free
            X[1:] = S.to_paper(x0[a - 1:n_hi])
            Xo, _ = S.iterate(X, S.coefs(np.zeros(L), a, L), K, precond, omega, history=False)
            xo = np.stack([S.from_paper(v) for v in Xo[1 + n_lo - a:]])
            xg = g.solution(n_lo, n_hi - n_lo + 1)
            assert field_errors(xg, xo, 2).max() < TOL, (n_lo, field_errors(xg, xo, 2))
    finally:
        g.close()


def test_trig_parity_ell_renumbered():
    """The §4.1 problem on a randomly renumbered mesh: the generic explicit-column (ELL)
    kernel with four load terms (sources and the lifting follow the renumbering)."""
    nt, K = 24, 8
    prob = trig_problem(4, nt, 1.0 / 64)
    perm = np.random.default_rng(3).permutation(prob.coords.shape[0])
    inv = np.argsort(perm)
    prob.coords = prob.coords[perm]
    prob.cells = inv[prob.cells].astype(np.int32)
    prob.dirichlet = prob.dirichlet.reshape(-1, 3)[perm].reshape(-1).copy()
    prob.dirichlet_values = prob.dirichlet_values.reshape(-1, 3)[perm].reshape(-1).copy()
    prob.x_initial = prob.x_initial.reshape(-1, 3)[perm].reshape(-1).copy()
    x0 = _x0(prob, nt)
    g = BiotSolver(prob, n_t=nt, precond=2, omega=0.5)
    try:
        assert g.info.kernel_path == 2
        g.set_iterate(1, x0)
        g.iterate(K)
        xg = g.solution()
        hg = np.stack([g.residual_history(kk) for kk in range(K)])
    finally:
        g.close()
    S, C, X = _oracle_start(prob, nt, x0)
    Xo, ho = S.iterate(X, C, K, 2, 0.5)
    xo = np.stack([S.from_paper(v) for v in Xo[1:]])
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


def test_sources_and_lifting_3d_parity():
    """Time-dependent sources and Dirichlet data on a 3D Kuhn mesh (column Dirichlet set,
    the 4-point quadrature, the generic kernel with four load terms)."""
    from workloads import make_problem
    nt, K = 20, 6
    prob = make_problem(3, 4, nt, 1.0 / nt, K, storage=1e-3, kappa_median=1e-2)
    prob.traction = np.zeros(3)

    def fn(q, xyz):
        out = np.zeros((xyz.shape[0], 4))
        if q == 0:
            out[:, 0] = np.sin(2 * xyz[:, 0])
            out[:, 1] = np.cos(xyz[:, 1]) * xyz[:, 2]
            out[:, 2] = xyz[:, 0] * xyz[:, 1]
        else:
            out[:, 3] = 1.0 + xyz[:, 0] ** 2 - xyz[:, 2]
        return out
    t = np.arange(nt + 1) / nt
    prob.source_fn = fn
    prob.n_sources = 2
    prob.source_coef = np.stack([np.cos(t[1:]), 1.0 + t[1:]])
    X3 = prob.coords
    prob.dirichlet_values = np.stack([X3[:, 0] * X3[:, 2], -X3[:, 1], 0.5 * X3[:, 2], 1.0 - X3[:, 2]], axis=1).reshape(-1)
    prob.dirichlet_coef = 1.0 + 0.5 * np.sin(3 * t)
    x0 = initial_iterate(prob.dirichlet, np.arange(1, nt + 1), 5)
    g = BiotSolver(prob, n_t=nt, precond=2, omega=0.5)
    try:
        assert g.info.kernel_path == 1
        g.set_iterate(1, x0)
        g.iterate(K)
        xg = g.solution()
        hg = np.stack([g.residual_history(kk) for kk in range(K)])
    finally:
        g.close()
    S = oracle.OracleSystem(prob)
    C = S.coefs(np.zeros(nt), 1, nt)
    X = np.zeros((nt + 1, S.ndof))
    X[1:] = S.to_paper(x0)
    Xo, ho = S.iterate(X, C, K, 2, 0.5)
    xo = np.stack([S.from_paper(v) for v in Xo[1:]])
    assert field_errors(xg, xo, 3).max() < TOL
    assert norm_errors(hg, ho).max() < TOL
