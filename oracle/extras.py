"""Oracle-only extras (TEST INFRASTRUCTURE ONLY; tiny sizes, scipy).

* sequential_be     -- Algorithm 1 with an exact (direct) solve per step
                       (P:L272-284): the fixed point the inverted scheme must
                       reach ("exactly consistent with the backward
                       Euler ... when N_thread = 1").
* iteration_matrix  -- dense I - omega P^{-1} AA for exact or diagonal P~1/P~2
                       (P:L238-262), used for the negative control (the
                       undamped literal iteration diverges, R1/R3).
* terzaghi_p / terzaghi_uy -- textbook 1-D consolidation closed form
                       (drained top, impermeable bottom, constrained modulus
                       lambda + 2 mu, storage S), the physics pin.
* gauss_seidel_in_time -- Algorithm 2 read literally with X^{n-1,m},
                       kept for the time-coupling pins.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla
import scipy.sparse.linalg as spla


def sequential_be(sysm, x0, s, nt):
    """Backward Euler, exact solve per step: AA x_n = A' x_{n-1} + s_n f (free DoFs).

    x0: paper-order x_0.  Returns X [(nt+1), ndof] paper order.
    """
    free = sysm.free > 0
    Aff = sysm.AA[free][:, free].tocsc()
    lu = spla.splu(Aff)
    X = np.zeros((nt + 1, sysm.ndof))
    X[0] = x0
    for n in range(1, nt + 1):
        b = sysm.AP @ X[n - 1] + sysm.load_vec(s, n)
        X[n, free] = lu.solve(b[free])
    return X


def iteration_matrix(sysm, precond=2, exact=True, omega=1.0):
    """Dense E = I - omega P^{-1} AA on the free DoFs (one time step)."""
    free = sysm.free > 0
    AA = sysm.AA[free][:, free].toarray()
    nu = int(free[:sysm.nu].sum())
    A = AA[:nu, :nu]
    BT = AA[nu:, :nu]
    St = -AA[nu:, nu:]
    if not exact:
        A = np.diag(np.diag(A))
        St = np.diag(np.diag(St))
    P = np.zeros_like(AA)
    P[:nu, :nu] = A
    P[nu:, nu:] = -St
    if precond == 1:
        P[nu:, :nu] = BT
    return np.eye(AA.shape[0]) - omega * sla.solve(P, AA)


def spectral_radius(E):
    return float(np.max(np.abs(np.linalg.eigvals(E))))


def terzaghi_p(y, t, lam, mu, alpha, S, kappa, L=1.0, sigma0=1.0, terms=400):
    """Pore pressure of 1-D consolidation, drained at y=L, impermeable at y=0.

    p0 = alpha sigma0 / (alpha^2 + S Mc), c_v = kappa / (S + alpha^2/Mc),
    p = sum_m 4 p0/((2m+1) pi) sin(k_m (L-y)) exp(-k_m^2 c_v t),
    k_m = (2m+1) pi / (2L), Mc = lambda + 2 mu.
    """
    Mc = lam + 2 * mu
    p0 = alpha * sigma0 / (alpha ** 2 + S * Mc)
    cv = kappa / (S + alpha ** 2 / Mc)
    y = np.asarray(y, dtype=np.float64)
    out = np.zeros_like(y)
    for m in range(terms):
        km = (2 * m + 1) * math.pi / (2 * L)
        out += 4 * p0 / ((2 * m + 1) * math.pi) * np.sin(km * (L - y)) * math.exp(-km * km * cv * t)
    return out


def terzaghi_uy(y, t, lam, mu, alpha, S, kappa, L=1.0, sigma0=1.0, terms=400):
    """Vertical displacement u_y = (alpha int_0^y p ds - sigma0 y) / Mc (fixed bottom)."""
    Mc = lam + 2 * mu
    p0 = alpha * sigma0 / (alpha ** 2 + S * Mc)
    cv = kappa / (S + alpha ** 2 / Mc)
    y = np.asarray(y, dtype=np.float64)
    ip = np.zeros_like(y)
    for m in range(terms):
        km = (2 * m + 1) * math.pi / (2 * L)
        c = 4 * p0 / ((2 * m + 1) * math.pi) * math.exp(-km * km * cv * t)
        ip += c * (np.cos(km * (L - y)) - math.cos(km * L)) / km
    return (alpha * ip - sigma0 * y) / Mc


def gauss_seidel_in_time(sysm, X, s, K, precond=2, omega=0.5, history=False):
    """Algorithm 2 literally: b^{n,m} uses X^{n-1,m} of the current sweep.

    history=True also returns the norms of the residual each update uses,
    r = A' X^{n-1,m} + f^n - AA X^{n,m-1}, split (u, p) as in R12: [K, nt, 2].
    """
    X = np.array(X, dtype=np.float64, copy=True)
    nt = X.shape[0] - 1
    nu = sysm.nu
    hist = np.zeros((K, nt, 2))
    for m in range(K):
        for n in range(1, nt + 1):
            r = sysm.AP @ X[n - 1] + sysm.load_vec(s, n) - sysm.AA @ X[n]
            hist[m, n - 1] = np.linalg.norm(r[:nu]), np.linalg.norm(r[nu:])
            z = np.empty_like(r)
            z[:nu] = sysm.DAinv * r[:nu]
            if precond == 2:
                z[nu:] = -sysm.DSinv * r[nu:]
            else:
                z[nu:] = sysm.DSinv * (sysm.BT @ z[:nu] - r[nu:])
            X[n] = X[n] + omega * z
    return (X, hist) if history else X

