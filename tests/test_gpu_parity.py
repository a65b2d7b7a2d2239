"""GPU (libbiot_pit.so, sm_100a) vs oracle parity -- needs a B200.

Tolerance: 1e-9 max relative error per field (BASELINE.json north star,
normwise per reading R17) on x^K, the fused residual history and the
residual norms at x^K.  Inputs: seeded x^0 ~ N(0,1) on free DoFs and
s_n = 1 + 0.1 sin n (DESIGN.md input recipe), both preconditioners and two
values of omega.
"""
import numpy as np
import pytest

import oracle
from paper_2310_10430_b200 import BiotSolver, FLAG_MANUAL_HALO
from workloads import config_problem, make_problem, initial_iterate, load_scales

from _parity import TOL, field_errors, norm_errors, subbox, oracle_window

pytestmark = pytest.mark.gpu


def _x0(prob, steps):
    return initial_iterate(prob.dirichlet, steps, prob.x0_seed)


def _run_full(prob, K, precond, omega, nt=None):
    nt = prob.n_t if nt is None else nt
    s = load_scales(nt, parity=True)
    x0 = _x0(prob, np.arange(1, nt + 1))
    g = BiotSolver(prob, n_t=nt, precond=precond, omega=omega, load_scale=s)
    g.set_iterate(1, x0)
    g.iterate(K)
    xg = g.solution()
    hg = np.stack([g.residual_history(k) for k in range(K)])
    rg = g.residual_norms()
    xo, ho, S = oracle.run(prob, x0, s, K, precond, omega)
    ro = S.residual_norms(np.vstack([np.zeros(S.ndof), S.to_paper(xo)]), s)
    return (xg, hg, rg), (xo, ho, ro)


@pytest.mark.parametrize("precond", [2, 1])
@pytest.mark.parametrize("omega", [0.5, 0.3])
def test_parity_config1_full(precond, omega):
    prob = config_problem(1)
    (xg, hg, rg), (xo, ho, ro) = _run_full(prob, prob.K, precond, omega)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL
    assert norm_errors(rg, ro).max() < TOL


@pytest.mark.parametrize("precond,omega,K", [(2, 0.5, 100), (1, 0.3, 20)])
def test_parity_config2_full(precond, omega, K):
    prob = config_problem(2)
    (xg, hg, rg), (xo, ho, ro) = _run_full(prob, K, precond, omega)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL
    assert norm_errors(rg, ro).max() < TOL


def _windows(nt, K, world=8, w=12):
    """Step windows covering the first/last K+8 steps and every 8-GPU slab boundary."""
    slab = nt // world
    wins = [(1, min(nt, K + 8)), (max(1, nt - K - 7), nt)]
    for r in range(1, world):
        b = r * slab
        wins.append((b - w // 2 + 1, b + w // 2))
    return wins


def _gpu_windowed(prob, K, precond, omega, wins):
    nt = prob.n_t
    s = load_scales(nt, parity=True)
    g = BiotSolver(prob, precond=precond, omega=omega, load_scale=s)
    for (a, b) in wins:
        lo = max(1, a - K)
        g.set_iterate(lo, _x0(prob, np.arange(lo, b + 1)))
    g.iterate(K)
    return g, s


@pytest.mark.parametrize("precond", [2, 1])
def test_parity_config3_windows(precond):
    """2D 512^2, N_t=1024 at full size; oracle on space-time windows (whole mesh)."""
    prob = config_problem(3)
    K, omega = 6, 0.5 if precond == 2 else 0.3
    wins = _windows(prob.n_t, K)
    g, s = _gpu_windowed(prob, K, precond, omega, wins)
    try:
        S = oracle.OracleSystem(prob)
        for (a, b) in wins:
            xo = oracle_window(S, lambda st: _x0(prob, st), s, a, b, K, precond, omega)
            xg = g.solution(a, b - a + 1)
            assert field_errors(xg, xo, 2).max() < TOL, (a, b)
    finally:
        g.close()


def _box_check(prob, g, s, K, precond, omega, lo, hi, wins, x0cache):
    sub, nodes, idx = subbox(prob, lo, hi)
    S = oracle.OracleSystem(sub)
    d, nc = prob.dim, prob.dim + 1
    n = prob.n
    # exact region: graph distance > reach*K from every cut face of the box; one
    # iteration reaches one node ring with P~2 and two with P~1 (B^T z_u gathers z_u,
    # itself a residual of the neighbours)
    reach = K * (2 if precond == 1 else 1)
    ok = np.ones(nodes.size, bool)
    for k in range(d):
        if lo[k] > 0:
            ok &= idx[:, k] > lo[k] + reach
        if hi[k] < n:
            ok &= idx[:, k] < hi[k] - reach
    assert ok.sum() > 0
    cols = (nodes[ok][:, None] * nc + np.arange(nc)).ravel()
    subcols = (np.nonzero(ok)[0][:, None] * nc + np.arange(nc)).ravel()
    for (a, b) in wins:
        full = x0cache[(a, b)]            # x^0 of steps max(1,a-K)..b, whole mesh
        first = max(1, a - K)
        x0f = lambda st: full[st - first].reshape(len(st), -1, nc)[:, nodes, :].reshape(len(st), -1)
        xo = oracle_window(S, x0f, s, a, b, K, precond, omega)
        xg = g.solution(a, b - a + 1)
        assert field_errors(xg[:, cols], xo[:, subcols], d).max() < TOL, (lo, hi, a, b)


@pytest.mark.parametrize("cid", [4, 5])
def test_parity_3d_spacetime_windows(cid):
    """3D configs at full size; oracle on space-time boxes (corner at the loaded top,
    an interior box, and the fixed bottom), windows at slab boundaries."""
    prob = config_problem(cid)
    K, precond, omega = 4, 2, 0.5
    wins = _windows(prob.n_t, K, w=8)
    if cid == 5:
        wins = wins[:3]
    g, s = _gpu_windowed(prob, K, precond, omega, wins)
    n = prob.n
    m = 2 * K + 6
    boxes = [((n - m, n - m, n - m), (n, n, n)),
             ((n // 2 - m // 2,) * 3, (n // 2 + m // 2,) * 3),
             ((0, 0, 0), (m, m, m))]
    try:
        x0cache = {(a, b): _x0(prob, np.arange(max(1, a - K), b + 1)) for (a, b) in wins}
        for lo, hi in boxes:
            _box_check(prob, g, s, K, precond, omega, np.array(lo), np.array(hi), wins, x0cache)
    finally:
        g.close()          # config 5 holds ~150 GB: release it even when an assertion fails


def test_parity_config4_p1_box():
    prob = config_problem(4)
    K, precond, omega = 3, 1, 0.3
    wins = _windows(prob.n_t, K, w=6)[:3]
    g, s = _gpu_windowed(prob, K, precond, omega, wins)
    n, m = prob.n, 14
    try:
        x0cache = {(a, b): _x0(prob, np.arange(max(1, a - K), b + 1)) for (a, b) in wins}
        _box_check(prob, g, s, K, precond, omega, np.array((n - m,) * 3), np.array((n,) * 3), wins,
                   x0cache)
    finally:
        g.close()


def test_parity_ell_path_renumbered_mesh():
    """A randomly renumbered mesh takes the explicit-column (ELL) kernel."""
    prob = make_problem(2, 12, 16, 1 / 16, 10, storage=1e-3, kappa_median=1e-2, x0_seed=4)
    perm = np.random.default_rng(0).permutation(prob.coords.shape[0])
    inv = np.argsort(perm)
    prob.coords = prob.coords[perm]
    prob.cells = inv[prob.cells].astype(np.int32)
    prob.facets = inv[prob.facets].astype(np.int32)
    prob.dirichlet = prob.dirichlet.reshape(-1, 3)[perm].reshape(-1).copy()
    for pc in (1, 2):
        (xg, hg, rg), (xo, ho, ro) = _run_full(prob, 10, pc, 0.5)
        assert field_errors(xg, xo, 2).max() < TOL
        assert norm_errors(hg, ho).max() < TOL


@pytest.mark.parametrize("dim", [2, 3])
def test_parity_ragged_and_small(dim):
    """n_t not a multiple of the 128-step warp chunk (ragged tail), N_t = 1, tiny meshes."""
    for nt in (1, 5, 130):
        prob = make_problem(dim, 3 if dim == 3 else 5, nt, 0.01, 7, x0_seed=8)
        (xg, hg, rg), (xo, ho, ro) = _run_full(prob, 7, 2, 0.5)
        assert field_errors(xg, xo, dim).max() < TOL, nt
        assert norm_errors(hg, ho).max() < TOL, nt


# ---- Gauss-Seidel in time (Alg. 2 literal) ----

def _gs_pair(prob, nt, K, precond, omega):
    from oracle import extras
    s = load_scales(nt, parity=True)
    x0 = _x0(prob, np.arange(1, nt + 1))
    g = BiotSolver(prob, n_t=nt, precond=precond, omega=omega, load_scale=s)
    try:
        g.set_iterate(1, x0)
        g.iterate_gs(K)
        xg = g.solution()
        hg = np.stack([g.residual_history(k) for k in range(K)])
    finally:
        g.close()
    S = oracle.OracleSystem(prob)
    X = np.zeros((nt + 1, S.ndof))
    X[1:] = S.to_paper(x0)
    Xo, ho = extras.gauss_seidel_in_time(S, X, s, K, precond, omega, history=True)
    return (xg, hg), (np.stack([S.from_paper(v) for v in Xo[1:]]), ho)


@pytest.mark.parametrize("precond,omega", [(2, 0.5), (1, 0.3)])
@pytest.mark.parametrize("nt,K", [(32, 6), (5, 9), (40, 40)])
def test_gs_parity_config1(precond, omega, nt, K):
    """Wavefront GS on the GPU vs the oracle's literal Algorithm 2: x^K and the residual
    of every (sweep, step) update; windows shorter and longer than K, N_t < K."""
    prob = config_problem(1)
    (xg, hg), (xo, ho) = _gs_pair(prob, nt, K, precond, omega)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


def test_gs_parity_config2_windows_span_chunks():
    """N_t = 256 with the lognormal-kappa 128^2 mesh: every wave runs the full tile grid."""
    prob = config_problem(2)
    (xg, hg), (xo, ho) = _gs_pair(prob, 256, 3, 2, 0.5)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


def test_gs_additive_and_converges_faster():
    """iterate_gs(a); iterate_gs(b) == iterate_gs(a + b) bitwise; after the same number of
    sweeps GS is closer to the backward-Euler solution than Jacobi (config 1)."""
    prob = config_problem(1)
    nt = prob.n_t
    s = load_scales(nt, parity=True)
    x0 = _x0(prob, np.arange(1, nt + 1))
    res = []
    for split in ((3, 4), (7,)):
        g = BiotSolver(prob, precond=2, omega=0.5, load_scale=s)
        g.set_iterate(1, x0)
        for k in split:
            g.iterate_gs(k)
        res.append((g.solution(), [g.residual_history(k) for k in range(7)]))
        g.close()
    assert np.array_equal(res[0][0], res[1][0])
    assert all(np.array_equal(a, b) for a, b in zip(res[0][1], res[1][1]))
    gj = BiotSolver(prob, precond=2, omega=0.5, load_scale=s)
    gj.set_iterate(1, x0)
    gj.iterate(7)
    gg = BiotSolver(prob, precond=2, omega=0.5, load_scale=s)
    gg.set_iterate(1, x0)
    gg.iterate_gs(7)
    assert (np.sqrt((gg.residual_norms() ** 2).sum()) < np.sqrt((gj.residual_norms() ** 2).sum()))
    gj.close()
    gg.close()


def test_gs_parity_long_windows():
    """K = 150 sweeps over N_t = 200: waves up to 150 steps wide run two 128-step chunks,
    the second taking q(t0-1) from the carry of the first."""
    prob = config_problem(1)
    (xg, hg), (xo, ho) = _gs_pair(prob, 200, 150, 2, 0.5)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


@pytest.mark.parametrize("precond,omega", [(2, 0.5), (1, 0.3)])
def test_gs_parity_3d(precond, omega):
    """3D tile kernel in wavefront GS (lognormal kappa, ragged windows) vs Alg. 2 literal."""
    prob = make_problem(3, 7, 40, 0.01, 6, storage=1e-3, kappa_median=1e-3, kappa_sigma=1.0,
                        kappa_seed=3, x0_seed=9)
    (xg, hg), (xo, ho) = _gs_pair(prob, 40, 7, precond, omega)
    assert field_errors(xg, xo, 3).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


# ---- per-step GMRES (Alg. 3 with K = GMRES) ----

def _gmres_pair(prob, nt, K, k, precond=2):
    from oracle import gmres as ogm
    s = load_scales(nt, parity=True)
    x0 = _x0(prob, np.arange(1, nt + 1))
    g = BiotSolver(prob, n_t=nt, precond=precond, omega=0.5, load_scale=s)
    try:
        g.set_iterate(1, x0)
        g.iterate_gmres(K, k)
        xg = g.solution()
        hg = np.stack([g.residual_history(kk) for kk in range(K)])
    finally:
        g.close()
    S = oracle.OracleSystem(prob)
    X = np.zeros((nt + 1, S.ndof))
    X[1:] = S.to_paper(x0)
    Xo, ho = ogm.iterate(S, X, s, K, k, precond=precond)
    return (xg, hg), (np.stack([S.from_paper(v) for v in Xo[1:]]), ho)


@pytest.mark.parametrize("nt,K,k", [(32, 3, 2), (40, 2, 5), (7, 3, 10)])
def test_gmres_parity_config1(nt, K, k):
    """One GMRES(k) cycle per step and outer iteration (CGS2 Arnoldi on the GPU, MGS in the
    oracle) vs the oracle's Alg. 3: x^K and the residual history at 1e-9."""
    prob = config_problem(1)
    (xg, hg), (xo, ho) = _gmres_pair(prob, nt, K, k)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


def test_gmres_parity_config2():
    prob = config_problem(2)
    (xg, hg), (xo, ho) = _gmres_pair(prob, 64, 2, 4)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


def _gs_gmres_pair(prob, nt, K, k, precond=2):
    from oracle import gmres as ogm
    s = load_scales(nt, parity=True)
    x0 = _x0(prob, np.arange(1, nt + 1))
    g = BiotSolver(prob, n_t=nt, precond=precond, omega=0.5, load_scale=s)
    try:
        g.set_iterate(1, x0)
        g.iterate_gs_gmres(K, k)
        xg = g.solution()
        hg = np.stack([g.residual_history(kk) for kk in range(K)])
    finally:
        g.close()
    S = oracle.OracleSystem(prob)
    X = np.zeros((nt + 1, S.ndof))
    X[1:] = S.to_paper(x0)
    Xo, ho = ogm.iterate(S, X, s, K, k, gauss_seidel=True, precond=precond)
    return (xg, hg), (np.stack([S.from_paper(v) for v in Xo[1:]]), ho)


@pytest.mark.parametrize("nt,K,k", [(32, 3, 4), (5, 7, 3)])
def test_gs_gmres_parity_config1(nt, K, k):
    """Alg. 3 literally (Gauss-Seidel in time, GMRES(k) per step) on the wavefront vs the
    oracle: x^K and every update's residual at 1e-9."""
    prob = config_problem(1)
    (xg, hg), (xo, ho) = _gs_gmres_pair(prob, nt, K, k)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


def test_gs_gmres_exact_solves_are_backward_euler_in_one_sweep():
    """with exact per-step solves (k >= the free DoFs) ONE Gauss-Seidel sweep of
    Alg. 3 is the sequential backward-Euler solution (checked on the GPU)."""
    from oracle import extras
    prob = make_problem(2, 2, 6, 1.0 / 6, 1, storage=1e-3, kappa_median=1e-2)
    S = oracle.OracleSystem(prob)
    assert (S.free > 0).sum() <= 16
    s = load_scales(6, parity=True)
    g = BiotSolver(prob, precond=2, omega=0.5, load_scale=s)
    try:
        g.iterate_gs_gmres(1, 16)
        xg = g.solution()
    finally:
        g.close()
    Xbe = extras.sequential_be(S, np.zeros(S.ndof), s, 6)
    xbe = np.stack([S.from_paper(v) for v in Xbe[1:]])
    assert field_errors(xg, xbe, 2).max() < 1e-9


@pytest.mark.parametrize("gs", [False, True])
def test_gmres_parity_3d(gs):
    """Per-step GMRES on the 3D tile kernel (ZOUT / MATVEC plane-march modes, 4D tensor
    maps of the Krylov panels): Jacobi and Gauss-Seidel in time vs the oracle's Alg. 3."""
    prob = make_problem(3, 6, 20, 1.0 / 20, 1, storage=1e-3, kappa_median=1e-3, kappa_sigma=1.0, kappa_seed=2)
    (xg, hg), (xo, ho) = (_gs_gmres_pair if gs else _gmres_pair)(prob, 20, 2, 4)
    assert field_errors(xg, xo, 3).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


# ---- per-step GMRES left-preconditioned by P~1 (eq. p1; the paper's §4.1 / §4.3 choice) ----

@pytest.mark.parametrize("nt,K,k", [(32, 3, 2), (7, 3, 10), (150, 2, 4)])
def test_gmres_p1_parity_config1(nt, K, k):
    """GMRES(k) per step with P~1 (tile ZOUT/MATVEC first half + the in-place z_p pass)
    vs the oracle's Alg. 3 with P~1: x^K and the residual history at 1e-9."""
    prob = config_problem(1)
    (xg, hg), (xo, ho) = _gmres_pair(prob, nt, K, k, precond=1)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


@pytest.mark.parametrize("gs", [False, True])
def test_gmres_p1_parity_3d(gs):
    prob = make_problem(3, 6, 20, 1.0 / 20, 1, storage=1e-3, kappa_median=1e-3, kappa_sigma=1.0, kappa_seed=2)
    (xg, hg), (xo, ho) = (_gs_gmres_pair if gs else _gmres_pair)(prob, 20, 2, 4, precond=1)
    assert field_errors(xg, xo, 3).max() < TOL
    assert norm_errors(hg, ho).max() < TOL


def test_gs_gmres_p1_parity_config1():
    prob = config_problem(1)
    (xg, hg), (xo, ho) = _gs_gmres_pair(prob, 32, 3, 4, precond=1)
    assert field_errors(xg, xo, 2).max() < TOL
    assert norm_errors(hg, ho).max() < TOL
