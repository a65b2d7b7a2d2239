"""Pins of the oracle's §4.1 loads (CPU only, no GPU).

* quadrature of the source loads: exact for the degrees the rules integrate (closed
  forms: int phi_a = |T|/(d+1) per cell; linear sources -> the consistent mass matrix);
* linear patch test: a solution affine in space and in time is reproduced EXACTLY by
  backward Euler with the sources and the Dirichlet lifting (every load term enters);
* the multi-term load keeps the fixed point: sequential BE is a fixed point of the
  inverted iteration with sources and lifting;
* PAPER.md Table 1 (loose, golden table1_trig.json): L2 error of p at t = 1 for
  h = 1/16, 1/32, 1/64 and its second-order decay.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import extras
from workloads import linear_patch_problem, trig_problem, patch_exact, trig_exact, make_problem

_GOLD = os.path.join(os.path.dirname(__file__), "golden", "table1_trig.json")

# L2 error quadrature (test side): the same published 7-point rule, restated here
_A1, _B1, _A2, _B2 = 0.059715871789770, 0.470142064105115, 0.797426985353087, 0.101286507323456
_QL = np.array([[1 / 3, 1 / 3, 1 / 3], [_A1, _B1, _B1], [_B1, _A1, _B1], [_B1, _B1, _A1],
                [_A2, _B2, _B2], [_B2, _A2, _B2], [_B2, _B2, _A2]])
_QW = np.array([0.225] + [0.132394152788506] * 3 + [0.125939180544827] * 3)


def l2_error_p(prob, p_nodal, t):
    X = prob.coords[prob.cells]
    E = X[:, 1:, :] - X[:, :1, :]
    area = np.abs(np.linalg.det(E)) / 2.0
    xq = np.einsum("ka,cad->ckd", _QL, X)
    ph = np.einsum("ka,ca->ck", _QL, p_nodal[prob.cells])
    pe = trig_exact(xq.reshape(-1, 2), t).reshape(ph.shape)
    return math.sqrt(float(np.sum(area[:, None] * _QW[None, :] * (ph - pe) ** 2)))


def full_field(prob, S, X, n):
    """Free part from the iteration + c_n x_D on the Dirichlet DoFs, node-interleaved."""
    fixed = np.asarray(prob.dirichlet, dtype=np.float64)
    return S.from_paper(X[n]) + prob.dirichlet_coef[n] * prob.dirichlet_values * fixed


def be_solution(prob):
    S = oracle.OracleSystem(prob)
    C = S.coefs(np.zeros(prob.n_t))
    x0 = S.to_paper(prob.x_initial) * S.free
    return S, C, extras.sequential_be(S, x0, C, prob.n_t)


@pytest.mark.parametrize("dim", [2, 3])
def test_quadrature_constant_and_linear(dim):
    """int 1 * phi_a summed = |Omega| = 1; linear f: the load equals M f_nodal (exact)."""
    prob = make_problem(dim, 3, 1, 0.1, 1)
    coords, cells = prob.coords, prob.cells
    bl = oracle.assemble_blocks(dim, coords, cells, 1.0, 1.0, 1.0, 1.0)
    ones = lambda q, xyz: np.ones((xyz.shape[0], dim + 1))
    F = oracle.source_load(dim, coords, cells, ones, 0, 0.5)
    nn = coords.shape[0]
    assert abs(F[:dim * nn].reshape(nn, dim)[:, 0].sum() - 1.0) < 1e-14
    assert abs(F[dim * nn:].sum() + 0.5) < 1e-14                 # -dt * |Omega|
    w = np.array([0.3, -1.1, 0.7, 0.2][:dim + 1])

    def lin(q, xyz):
        v = w[0] + xyz @ w[1:]
        return np.repeat(v[:, None], dim + 1, axis=1)
    F = oracle.source_load(dim, coords, cells, lin, 0, 1.0)
    fn = w[0] + coords @ w[1:]
    ref = bl.M @ fn
    assert np.abs(F[:dim * nn].reshape(nn, dim)[:, 0] - ref).max() < 1e-14
    assert np.abs(F[dim * nn:] + ref).max() < 1e-14


def test_quadrature_degree5_triangle():
    """The 2D rule integrates x^a y^b (a + b <= 4) times phi exactly: compare the single-
    cell load with the exact monomial integrals over the reference triangle."""
    coords = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    cells = np.array([[0, 1, 2]], dtype=np.int32)
    for a_, b_ in [(4, 0), (2, 2), (1, 3), (3, 1), (0, 4)]:
        fn = lambda q, xyz: np.repeat((xyz[:, 0] ** a_ * xyz[:, 1] ** b_)[:, None], 3, axis=1)
        F = oracle.source_load(2, coords, cells, fn, 0, 1.0)
        # phi_1 = x: int x^(a+1) y^b = (a+1)! b! / (a+b+3)!
        exact1 = math.factorial(a_ + 1) * math.factorial(b_) / math.factorial(a_ + b_ + 3)
        assert abs(F[2 * 1] - exact1) < 1e-15, (a_, b_)
        total = math.factorial(a_) * math.factorial(b_) / math.factorial(a_ + b_ + 2)
        assert abs(F[0] + F[2] + F[4] - total) < 1e-15


def test_linear_patch_exact():
    prob = linear_patch_problem(8, 12, 0.1)
    S, C, X = be_solution(prob)
    for n in range(prob.n_t + 1):
        ref = patch_exact(prob.coords, n * prob.dt)
        assert np.abs(full_field(prob, S, X, n) - ref).max() < 1e-12 * np.abs(ref).max()


def test_patch_lifting_terms_matter():
    """Negative control: dropping the A' lifting (previous Dirichlet values) breaks it."""
    prob = linear_patch_problem(6, 4, 0.1)
    S = oracle.OracleSystem(prob)
    C = S.coefs(np.zeros(prob.n_t))
    j = [k[0] for k in S.kinds].index("dprev")
    C[j] = 0.0
    X = extras.sequential_be(S, S.to_paper(prob.x_initial) * S.free, C, prob.n_t)
    ref = patch_exact(prob.coords, prob.n_t * prob.dt)
    assert np.abs(full_field(prob, S, X, prob.n_t) - ref).max() > 1e-3


@pytest.mark.parametrize("precond", [1, 2])
def test_trig_be_is_fixed_point(precond):
    prob = trig_problem(3, 16, 1 / 16)
    S, C, X = be_solution(prob)
    assert S.residual_norms(X, C).max() < 1e-12 * np.abs(S.Fall).max()
    X2, _ = S.iterate(X.copy(), C, 3, precond, 0.5, history=False)
    assert np.abs(X2 - X).max() < 1e-12 * np.abs(X).max()


def test_table1_trig_errors():
    gold = json.load(open(_GOLD))
    errs = []
    for row in gold["rows"]:
        prob = trig_problem(row["k"], int(round(gold["t"] / gold["tau"])), gold["tau"])
        S, C, X = be_solution(prob)
        p = full_field(prob, S, X, prob.n_t).reshape(-1, 3)[:, 2]
        e = l2_error_p(prob, p, gold["t"])
        lo, hi = row["band"]
        assert lo * row["l2_p"] <= e <= hi * row["l2_p"], (row, e)
        errs.append(e)
    # second-order decay in h on uniform meshes (superconvergence)
    for a, b in zip(errs, errs[1:]):
        assert 3.3 < a / b < 4.8, errs
