"""Pins of the oracle's discretisation (CPU only, no GPU).

Every check compares the oracle against something other than itself:
golden values (SPEC/PAPER, tests/golden/), closed-form integrals of linear
fields, kernels of the operators, and textbook stencils.  A dropped term,
wrong sign, wrong coefficient or transposed block fails at least one.
"""
import json
import os

import numpy as np
import pytest

import oracle
from workloads import make_problem, mesh_square, mesh_cube

GOLD = os.path.join(os.path.dirname(__file__), "golden", "lame_beta.json")


def test_lame_beta_golden():
    g = json.load(open(GOLD))
    for c in g["lame"]:
        lam, mu = oracle.lame(c["E"], c["nu"])
        assert abs(lam - c["lambda"]) <= c["tol"] * max(1, abs(c["lambda"])), c
        assert abs(mu - c["mu"]) <= c["tol"] * max(1, abs(c["mu"])), c
    for c in g["beta"]:
        if "E" in c:
            lam, mu = oracle.lame(c["E"], c["nu"])
        else:
            lam, mu = c["lambda"], c["mu"]
        b = oracle.beta(c["h"], lam, mu)
        assert abs(b - c["beta"]) <= c["tol"], (b, c)
    # beta is linear in h
    assert oracle.beta(0.5, 1.0, 1.0) == pytest.approx(2 * oracle.beta(0.25, 1.0, 1.0), rel=1e-15)


def _lin_strain_energy(G, lam, mu):
    eps = 0.5 * (G + G.T)
    return 2 * mu * np.sum(eps * eps) + lam * np.trace(eps) ** 2


@pytest.mark.parametrize("d", [2, 3])
def test_element_closed_forms(d):
    rng = np.random.default_rng(3)
    X = np.eye(d + 1, d, k=-1) if d == 2 else np.vstack([np.zeros(3), np.eye(3)])
    X = X + 0.1 * rng.standard_normal(X.shape)
    vol_ref = abs(np.linalg.det(X[1:] - X[0])) / (2 if d == 2 else 6)
    lam, mu, alpha = 0.7, 1.3, 0.9
    Ae, Be, Le, Me, vol = oracle.element(d, X, lam, mu, alpha)
    assert vol == pytest.approx(vol_ref, rel=1e-13)
    G = rng.standard_normal((d, d))      # linear field u(x) = G x
    u = (X @ G.T).reshape(-1)            # nodal values, (a, c) ordering
    assert u @ Ae @ u == pytest.approx(vol * _lin_strain_energy(G, lam, mu), rel=1e-12)
    g = rng.standard_normal(d)           # linear pressure p = g . x
    p = X @ g
    assert p @ Le @ p == pytest.approx(vol * g @ g, rel=1e-12)
    # mass: int p q over a simplex, p=q=1 -> |T|; exact for linear p (quadrature by
    # vertex+centroid formula for quadratics: int f = |T|/((d+1)(d+2)) (sum f_a f_b (1+delta)))
    assert Me.sum() == pytest.approx(vol, rel=1e-14)
    # B: sum_b (Be^T u)_b = -alpha int div u = -alpha |T| tr(G); each entry equal
    btu = Be.T @ u
    assert np.allclose(btu, -alpha * vol * np.trace(G) / (d + 1), rtol=1e-12, atol=0)


def _blocks(dim, n, lam=1.0, mu=1.0, alpha=1.0, kappa=1.0):
    coords, cells = mesh_square(n) if dim == 2 else mesh_cube(n)
    return coords, cells, oracle.assemble_blocks(dim, coords, cells, lam, mu, alpha,
                                                 np.full(cells.shape[0], kappa))


def test_laplacian_stencil_2d():
    """Interior row of L on the right-triangle mesh = 5-point stencil."""
    n = 4
    coords, cells, bl = _blocks(2, n)
    L = bl.L.toarray()
    assert np.allclose(L.sum(axis=1), 0, atol=1e-14)
    w = n + 1
    i = 2 * w + 2
    row = L[i]
    assert row[i] == pytest.approx(4.0, abs=1e-14)
    for off in (1, -1, w, -w):
        assert row[i + off] == pytest.approx(-1.0, abs=1e-14)
    for off in (w + 1, -w - 1):               # structural but zero on this mesh
        assert abs(row[i + off]) < 1e-14
    assert np.count_nonzero(np.abs(row) > 1e-14) == 5


def test_laplacian_stencil_3d():
    """Interior row of L on the Kuhn mesh = 7-point stencil 6h, -h."""
    n = 3
    h = 1.0 / n
    coords, cells, bl = _blocks(3, n)
    L = bl.L.toarray()
    assert np.allclose(L.sum(axis=1), 0, atol=1e-14)
    w = n + 1
    i = (1 * w + 1) * w + 1
    row = L[i]
    assert row[i] == pytest.approx(6 * h, abs=1e-14)
    for off in (1, w, w * w):
        assert row[i + off] == pytest.approx(-h, abs=1e-14)
        assert row[i - off] == pytest.approx(-h, abs=1e-14)
    assert np.count_nonzero(np.abs(row) > 1e-14) == 7
    # 15 structural neighbours (Kuhn): 14 + self
    assert bl.L[i].nnz == 15


@pytest.mark.parametrize("dim,n", [(2, 3), (3, 2)])
def test_elasticity_kernel_and_energy(dim, n):
    lam, mu = 0.8, 1.7
    coords, cells, bl = _blocks(dim, n, lam=lam, mu=mu)
    A = bl.A.toarray()
    assert np.abs(A - A.T).max() < 1e-13
    nn = coords.shape[0]
    # rigid translations and infinitesimal rotations
    for c in range(dim):
        t = np.zeros((nn, dim)); t[:, c] = 1
        assert np.abs(A @ t.ravel()).max() < 1e-12
    pairs = [(0, 1)] if dim == 2 else [(0, 1), (0, 2), (1, 2)]
    for a, b in pairs:
        r = np.zeros((nn, dim)); r[:, a] = -coords[:, b]; r[:, b] = coords[:, a]
        assert np.abs(A @ r.ravel()).max() < 1e-12
    # strain energy of a linear field over the unit domain (|Omega| = 1)
    G = np.random.default_rng(1).standard_normal((dim, dim))
    u = (coords @ G.T).ravel()
    assert u @ A @ u == pytest.approx(_lin_strain_energy(G, lam, mu), rel=1e-12)


@pytest.mark.parametrize("dim,n", [(2, 4), (3, 2)])
def test_coupling_mass_diffusion(dim, n):
    alpha = 0.6
    coords, cells, bl = _blocks(dim, n, alpha=alpha)
    _, _, bl2 = _blocks(dim, n, alpha=2 * alpha)
    assert np.abs(bl2.B.toarray() - 2 * bl.B.toarray()).max() < 1e-15
    nn = coords.shape[0]
    G = np.random.default_rng(2).standard_normal((dim, dim))
    u = (coords @ G.T).ravel()
    one = np.ones(nn)
    # B^T u_lin = -alpha tr(G) M 1  (div u constant; int phi_q div u = tr(G) (M 1)_q)
    assert np.allclose(bl.B.T @ u, -alpha * np.trace(G) * (bl.M @ one), rtol=0, atol=1e-13)
    # mass integrals of linear fields over the unit domain
    assert one @ bl.M @ one == pytest.approx(1.0, rel=1e-14)
    x, y = coords[:, 0], coords[:, 1]
    assert x @ bl.M @ y == pytest.approx(0.25, rel=1e-13)
    assert x @ bl.M @ x == pytest.approx(1.0 / 3.0, rel=1e-13)
    # heterogeneous kappa: p^T C p = |grad p|^2 sum_e kappa_e |T_e| for linear p
    kap = np.random.default_rng(5).uniform(0.5, 2.0, cells.shape[0])
    bk = oracle.assemble_blocks(dim, coords, cells, 1.0, 1.0, 1.0, kap)
    g = np.arange(1, dim + 1, dtype=float)
    p = coords @ g
    vols = 1.0 / cells.shape[0]
    assert p @ bk.C @ p == pytest.approx(g @ g * np.sum(kap * vols), rel=1e-12)
    assert np.abs((bl.C - bl.L).toarray()).max() < 1e-15     # kappa = 1 -> C = L


@pytest.mark.parametrize("dim,n", [(2, 8), (3, 3)])
def test_traction_load(dim, n):
    prob = make_problem(dim, n, 2, 0.5, 1)
    F = oracle.traction_load(dim, prob.coords, prob.facets, prob.traction).reshape(-1, dim)
    assert F[:, dim - 1].sum() == pytest.approx(-1.0, rel=1e-14)    # unit load on unit top
    assert np.abs(F[:, :dim - 1]).max() == 0.0
    if dim == 2:
        h = 1.0 / n
        w = n + 1
        top = np.arange(n * w, w * w)
        assert F[top[1], 1] == pytest.approx(-h, rel=1e-14)
        assert F[top[0], 1] == pytest.approx(-h / 2, rel=1e-14)


def _free_sys(dim, n, storage=0.3, dt=0.05, kappa=0.7, lam=1.1, mu=0.9, alpha=0.8):
    prob = make_problem(dim, n, 2, dt, 1, lam=lam, mu=mu, alpha=alpha, storage=storage,
                        kappa_median=kappa)
    free = np.zeros_like(prob.dirichlet)
    return prob, oracle.OracleSystem(prob, dirichlet=free)


@pytest.mark.parametrize("dim,n", [(2, 4), (3, 2)])
def test_operator_composition_via_residual(dim, n):
    """r = A' x_prev + s f - AA x_cur against closed forms (pins AA and A' blocks)."""
    prob, S = _free_sys(dim, n)
    nn = S.nn
    coords = prob.coords
    g = np.linspace(0.5, 1.5, dim)
    p_lin = coords @ g
    G = np.random.default_rng(7).standard_normal((dim, dim))
    u_lin = (coords @ G.T).ravel()
    zero_u = np.zeros(S.nu)
    s0 = np.zeros(1)
    beta = oracle.beta(prob.h, prob.lam, prob.mu)

    def res(x_prev, x_cur, s=s0):
        X = np.stack([x_prev, x_cur])
        _, r = S.residual_norms(X, s, return_r=True)
        return r[0]

    # 1) x_prev = x_cur = (0, p_lin): r_p = (S~ - H) p = tau C p  -> p^T r_p = tau kappa |g|^2
    y = np.concatenate([zero_u, p_lin])
    r = res(y, y)
    assert p_lin @ r[S.nu:] == pytest.approx(prob.dt * 0.7 * g @ g, rel=1e-11)
    # 2) x_cur = 0, x_prev = (0, p_lin): r_p = -H p -> p^T r_p = -(S int p^2 + beta |g|^2)
    int_p2 = p_lin @ S.blocks.M @ p_lin
    r = res(y, np.zeros(S.ndof))
    assert p_lin @ r[S.nu:] == pytest.approx(-(prob.storage * int_p2 + beta * g @ g), rel=1e-11)
    assert np.abs(r[:S.nu]).max() == 0.0                    # A' has no displacement rows
    # 3) x_cur = (u_lin, 0): r_u = -A u, r_p = -B^T u
    xc = np.concatenate([u_lin, np.zeros(nn)])
    r = res(np.zeros(S.ndof), xc)
    assert u_lin @ r[:S.nu] == pytest.approx(-_lin_strain_energy(G, prob.lam, prob.mu), rel=1e-11)
    assert r[S.nu:].sum() == pytest.approx(prob.alpha * np.trace(G), rel=1e-11)
    # 4) x_cur = (0, 1): r_u = -B 1 -> u_lin^T r_u = -(B^T u_lin)^T 1 = alpha tr(G)
    xc = np.concatenate([zero_u, np.ones(nn)])
    r = res(np.zeros(S.ndof), xc)
    assert u_lin @ r[:S.nu] == pytest.approx(prob.alpha * np.trace(G), rel=1e-11)
    # 5) load: x = 0, s = 2 -> r = 2 f
    r = res(np.zeros(S.ndof), np.zeros(S.ndof), np.array([2.0]))
    F = oracle.traction_load(dim, prob.coords, prob.facets, prob.traction)
    assert np.allclose(r[:S.nu], 2 * F, rtol=0, atol=1e-15)
    # AA symmetric (P:L193-196 with B^T below B)
    assert abs(S.AA - S.AA.T).max() < 1e-13


def test_dirichlet_restriction():
    prob = make_problem(2, 4, 2, 0.1, 1)
    S = oracle.OracleSystem(prob)
    fixed = S.free == 0
    assert fixed.sum() == int(prob.dirichlet.sum())
    AA = S.AA.toarray()
    assert np.abs(AA[fixed]).max() == 0 and np.abs(AA[:, fixed]).max() == 0
    assert np.abs(S.F[fixed]).max() == 0
    assert np.all(S.DAinv[fixed[:S.nu]] == 0) and np.all(S.DSinv[fixed[S.nu:]] == 0)
    assert np.all(S.DAinv[~fixed[:S.nu]] > 0) and np.all(S.DSinv[~fixed[S.nu:]] > 0)
    # layout round trip (R20)
    x = np.random.default_rng(0).standard_normal(S.ndof)
    assert np.array_equal(S.from_paper(S.to_paper(x)), x)
    # u_x of node k lives at interleaved index k*(d+1)
    xi = np.zeros(S.ndof); xi[5 * 3 + 1] = 1.0
    assert S.to_paper(xi)[5 * 2 + 1] == 1.0
