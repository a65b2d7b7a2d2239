"""Helpers for GPU-vs-oracle parity tests (test code only)."""
from __future__ import annotations

import numpy as np

import oracle
from workloads import initial_iterate
from workloads.generators import Problem

TOL = 1e-9   # BASELINE.json north star: 1e-9 max relative error per field (reading R17: normwise)


def field_errors(x, ref, dim):
    """Per field f in {u_1..u_d, p}: max|x - ref| / max|ref| over all steps and nodes."""
    nc = dim + 1
    a = np.asarray(x).reshape(-1, nc)
    b = np.asarray(ref).reshape(-1, nc)
    out = []
    for c in range(nc):
        den = np.abs(b[:, c]).max()
        num = np.abs(a[:, c] - b[:, c]).max()
        out.append(num / den if den > 0 else num)
    return np.array(out)


def norm_errors(h, href):
    """Per part (u, p): max_n |h - href| / max_n href."""
    h = np.asarray(h).reshape(-1, 2)
    r = np.asarray(href).reshape(-1, 2)
    out = []
    for k in range(2):
        den = np.abs(r[:, k]).max()
        out.append(np.abs(h[:, k] - r[:, k]).max() / den if den > 0 else np.abs(h[:, k]).max())
    return np.array(out)


def subbox(prob: Problem, lo, hi):
    """Sub-problem made of the cells inside the index box [lo, hi) (cells per axis).

    Returns (sub_problem, node_ids) where node_ids maps sub-node -> global node.
    Cells are kept in global orientation; Dirichlet DoFs and traction facets are
    the global ones restricted to the box (reading: the cut faces are *not*
    boundaries -- the values within graph distance K of a cut face are wrong
    after K iterations and must not be compared).
    """
    d, n = prob.dim, prob.n
    w = n + 1
    lo = np.asarray(lo); hi = np.asarray(hi)
    # node index vectors
    nid = np.arange(prob.coords.shape[0])
    idx = np.stack([(nid // w ** k) % w for k in range(d)], axis=1)
    inbox = np.all((idx >= lo) & (idx <= hi), axis=1)
    keep_cells = np.all(inbox[prob.cells], axis=1)
    nodes = np.nonzero(inbox)[0]
    g2l = -np.ones(prob.coords.shape[0], dtype=np.int64)
    g2l[nodes] = np.arange(nodes.size)
    cells = g2l[prob.cells[keep_cells]].astype(np.int32)
    fk = np.all(inbox[prob.facets], axis=1)
    facets = g2l[prob.facets[fk]].astype(np.int32)
    nc = d + 1
    dirichlet = prob.dirichlet.reshape(-1, nc)[nodes].reshape(-1).copy()
    kappa = prob.kappa[keep_cells]
    sub = Problem(dim=d, n=n, n_t=prob.n_t, dt=prob.dt, K=prob.K, lam=prob.lam, mu=prob.mu,
                  alpha=prob.alpha, storage=prob.storage, kappa=kappa, h=prob.h,
                  coords=prob.coords[nodes], cells=cells, dirichlet=dirichlet, facets=facets,
                  traction=prob.traction, x0_seed=prob.x0_seed, name=prob.name + "-box")
    return sub, nodes, idx[nodes]


def oracle_window(sysm, x0_fn, s, n_lo, n_hi, K, precond, omega, ghost=None, nthreads=0):
    """Oracle x^K for global steps [n_lo, n_hi] from a window starting at max(1, n_lo-K).

    x0_fn(steps) -> [len, ndof] node-interleaved x^0 of those global steps (sub-numbering).
    Returns [n_hi-n_lo+1, ndof] node-interleaved, exact by the light-cone argument.
    """
    a = max(1, n_lo - K)
    steps = np.arange(a, n_hi + 1)
    X = np.zeros((steps.size + 1, sysm.ndof))
    if ghost is not None and a > 1:
        X[0] = sysm.to_paper(ghost)
    X[1:] = sysm.to_paper(x0_fn(steps))
    X, _ = sysm.iterate(X, s[steps - 1], K, precond, omega, history=False, nthreads=nthreads)
    return sysm.from_paper(X[1 + (n_lo - a):])


def oracle_window_full(sysm, x0_fn, s, n_lo, n_hi, K, precond, omega, nthreads=0):
    """As oracle_window, plus the residual history and the norms at x^K.

    Returns (x [L, ndof], hist [K, L, 2], norms [L, 2], exact_from) for the global steps
    n_lo..n_hi (L = n_hi - n_lo + 1).  The oracle starts at a = max(1, n_lo - K) with a
    zero ghost; x^k_n is exact for n >= a + k (one step of the light cone per iteration),
    so x^K and every history entry r(x^k)_n (k < K) are exact on the window, and the norms
    at x^K from step exact_from on (n_lo + 1 when a > 1: r(x^K)_{n_lo} reads x^K_{n_lo-1};
    every step when a = 1, whose ghost is the true x_0).
    """
    a = max(1, n_lo - K)
    steps = np.arange(a, n_hi + 1)
    X = np.zeros((steps.size + 1, sysm.ndof))
    X[1:] = sysm.to_paper(x0_fn(steps))
    X, hist = sysm.iterate(X, s[steps - 1], K, precond, omega, history=True, nthreads=nthreads)
    rn = sysm.residual_norms(X, s[steps - 1], nthreads=nthreads)
    o = n_lo - a
    return (sysm.from_paper(X[1 + o:]), hist[:, o:], rn[o:], n_lo if a == 1 else n_lo + 1)
