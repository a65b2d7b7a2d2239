"""Chebyshev-Jacobi inner inverses for the block preconditioners (TEST INFRASTRUCTURE ONLY).

SURVEY §8(f) NEXT-1, reading R22: the paper's P~2 = [[A, 0], [0, -S~p]]
and P~1 = [[A, 0], [B^T, -S~p]] (PAPER.md eqs. p1/p2) need A^{-1} and
S~p^{-1}; the diagonal inverses of R2 are replaced by m steps of Chebyshev iteration
preconditioned by the diagonal (Saad, Iterative Methods for Sparse Linear Systems,
Alg. 12.1 with M -> D^{-1} M) on the interval [lambda_max / alpha, lambda_max] of
D^{-1} M, lambda_max = the Gershgorin bound max_i sum_j |M_ij| / M_ii.  m = 1 is the
diagonal inverse scaled by 1 / theta.

Only tests/ and bench.py's CPU legs use this module (as the rest of oracle/).
Pins: tests/test_oracle_chebyshev.py (closed-form Chebyshev polynomial on a diagonal
operator, convergence to the direct solve, the backward-Euler fixed point).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def gershgorin_max(M, Dinv):
    """Upper bound of the spectrum of D^{-1} M over the rows with Dinv != 0."""
    rows = np.asarray(abs(M).sum(axis=1)).ravel()
    v = rows * np.abs(Dinv)
    return float(v[Dinv != 0].max())


def chebyshev(M, Dinv, b, m, lmin, lmax):
    """m Chebyshev steps for M y = b from y_0 = 0, preconditioner D = diag(M).

    b: [n] or [n, k] (k right-hand sides, e.g. the time steps).  The recurrence
    (theta, delta the centre and half width of [lmin, lmax], sigma = theta / delta):
        r_0 = b, d_0 = D^{-1} r_0 / theta, y_1 = d_0,
        r_k = r_{k-1} - M d_{k-1},  rho_k = 1 / (2 sigma - rho_{k-1}),  rho_0 = 1 / sigma,
        d_k = rho_k rho_{k-1} d_{k-1} + (2 rho_k / delta) D^{-1} r_k,  y_{k+1} = y_k + d_k.
    """
    theta = 0.5 * (lmax + lmin)
    delta = 0.5 * (lmax - lmin)
    sigma = theta / delta
    Dc = Dinv if np.ndim(b) == 1 else Dinv[:, None]
    r = np.array(b, dtype=np.float64, copy=True)
    d = Dc * r / theta
    y = d.copy()
    rho = 1.0 / sigma
    for _ in range(1, m):
        r = r - M @ d
        rho_new = 1.0 / (2.0 * sigma - rho)
        d = rho_new * rho * d + (2.0 * rho_new / delta) * (Dc * r)
        rho = rho_new
        y = y + d
    return y


class ChebyshevPrecond:
    """Per-block Chebyshev data of an oracle.OracleSystem: A = AA[:nu, :nu],
    S~p = -AA[nu:, nu:] (Dirichlet rows/columns already removed), diagonals DAinv, DSinv."""

    def __init__(self, sysm, m, alpha=30.0):
        nu = sysm.nu
        self.m = m
        self.A = sysm.AA[:nu, :nu].tocsr()
        self.St = (-sysm.AA[nu:, nu:]).tocsr()
        self.lmax_u = gershgorin_max(self.A, sysm.DAinv)
        self.lmax_p = gershgorin_max(self.St, sysm.DSinv)
        self.alpha = alpha
        self.sysm = sysm

    def apply(self, R, precond=2):
        """Z = P~^{-1} R for R [nt, ndof] (paper order), inner inverses by Chebyshev."""
        S = self.sysm
        nu = S.nu
        Ru, Rp = R[:, :nu].T, R[:, nu:].T
        Zu = chebyshev(self.A, S.DAinv, Ru, self.m, self.lmax_u / self.alpha, self.lmax_u)
        if precond == 2:
            Zp = -chebyshev(self.St, S.DSinv, Rp, self.m, self.lmax_p / self.alpha, self.lmax_p)
        else:
            Zp = chebyshev(self.St, S.DSinv, S.BT @ Zu - Rp, self.m, self.lmax_p / self.alpha, self.lmax_p)
        return np.concatenate([Zu.T, Zp.T], axis=1)


def iterate(sysm, X, s, K, m, precond=2, omega=0.5, alpha=30.0):
    """K Jacobi-in-time outer iterations (R4) with Chebyshev inner inverses.

    X [(nt+1), ndof] paper order, X[0] the fixed previous state.  Returns (X, history)
    with history [K, nt, 2] the (u, p) norms of the residual at x^k (R12).
    """
    X = np.array(X, dtype=np.float64, copy=True)
    nt = X.shape[0] - 1
    nu = sysm.nu
    P = ChebyshevPrecond(sysm, m, alpha)
    hist = np.zeros((K, nt, 2))
    S, Fm = sysm._loadset(s)
    for k in range(K):
        R = (sysm.AP @ X[:-1].T).T + S.T @ Fm - (sysm.AA @ X[1:].T).T
        hist[k, :, 0] = np.linalg.norm(R[:, :nu], axis=1)
        hist[k, :, 1] = np.linalg.norm(R[:, nu:], axis=1)
        X[1:] += omega * P.apply(R, precond)
    return X, hist
