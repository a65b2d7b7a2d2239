"""Per-step GMRES inside the inverted time-stepping scheme (TEST INFRASTRUCTURE ONLY).

PAPER.md Alg. 3: X^{n,m} = K(P, AA, X^{n,m-1}, b^{n,m}, n_iter), K an
iterative solver with preconditioner P run for n_iter iterations per call; the paper's
solver is GMRES.  Reading R23: one cycle of GMRES(k),
k = n_iter, LEFT-preconditioned by the paper's block preconditioner with diagonal inner
inverses (P~2, eq. p2, or P~1, eq. p1 -- the paper's choice for §4.1 and §4.3, P:L523-524,
P:L826; the Arnoldi vectors span K_k(P^{-1} AA, P^{-1} r0) and the cycle minimises
||P^{-1}(b - AA x)||_2), per time
step, started from X^{n,m-1}; b^{n,m} = A' X^{n-1,m-1} + f^n (Jacobi in time, R4) or
A' X^{n-1,m} + f^n (Gauss-Seidel, Alg. 3 literal).  Arnoldi by modified Gram-Schmidt,
the small least-squares problem by numpy's lstsq (a library primitive).

Pins: tests/test_oracle_gmres.py.
"""
from __future__ import annotations

import numpy as np


def apply_p2inv(sysm, r):
    """z = P~2^{-1} r with diagonal inner inverses (R2): z_u = D_A^{-1} r_u, z_p = -D_S^{-1} r_p."""
    nu = sysm.nu
    z = np.empty_like(r)
    z[:nu] = sysm.DAinv * r[:nu]
    z[nu:] = -sysm.DSinv * r[nu:]
    return z


def apply_p1inv(sysm, r):
    """z = P~1^{-1} r, P~1 = [[A, 0], [B^T, -S~p]] (eq. p1) with diagonal inner
    inverses (R2): z_u = D_A^{-1} r_u, then B^T z_u - S~p z_p = r_p gives
    z_p = D_S^{-1} (B^T z_u - r_p)."""
    nu = sysm.nu
    z = np.empty_like(r)
    z[:nu] = sysm.DAinv * r[:nu]
    z[nu:] = sysm.DSinv * (sysm.BT @ z[:nu] - r[nu:])
    return z


def apply_pinv(sysm, r, precond=2):
    return apply_p2inv(sysm, r) if precond == 2 else apply_p1inv(sysm, r)


def gmres_cycle(sysm, x, b, k, precond=2):
    """One GMRES(k) cycle for AA x = b from x, left-preconditioned by P~precond.
    Returns (x_new, ||P^{-1} r0||, ||P^{-1} r_new||)."""
    AA = sysm.AA
    r0 = apply_pinv(sysm, b - AA @ x, precond)
    beta = np.linalg.norm(r0)
    if beta == 0.0:
        return x.copy(), 0.0, 0.0
    V = [r0 / beta]
    H = np.zeros((k + 1, k))
    kk = k
    for j in range(k):
        w = apply_pinv(sysm, AA @ V[j], precond)
        for i in range(j + 1):
            H[i, j] = V[i] @ w
            w = w - H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        if H[j + 1, j] == 0.0:          # lucky breakdown: the Krylov space is invariant
            kk = j + 1
            break
        V.append(w / H[j + 1, j])
    e1 = np.zeros(kk + 1)
    e1[0] = beta
    y = np.linalg.lstsq(H[:kk + 1, :kk], e1, rcond=None)[0]
    xn = x + np.column_stack(V[:kk]) @ y
    rn = np.linalg.norm(apply_pinv(sysm, b - AA @ xn, precond))
    return xn, beta, rn


def iterate(sysm, X, s, K, k, gauss_seidel=False, precond=2):
    """K outer iterations of Alg. 3 with per-step GMRES(k) (P~precond, left).

    X [(nt+1), ndof] paper order, X[0] the fixed previous state.  Returns (X, hist)
    with hist [K, nt, 2] the (u, p) norms of the unpreconditioned residual
    b^{n,m} - AA X^{n,m-1} each cycle starts from (R12)."""
    X = np.array(X, dtype=np.float64, copy=True)
    nt = X.shape[0] - 1
    nu = sysm.nu
    hist = np.zeros((K, nt, 2))
    for m in range(K):
        Xold = X.copy()
        for n in range(1, nt + 1):
            prev = X[n - 1] if gauss_seidel else Xold[n - 1]
            b = sysm.AP @ prev + sysm.load_vec(s, n)
            r = b - sysm.AA @ Xold[n]
            hist[m, n - 1] = np.linalg.norm(r[:nu]), np.linalg.norm(r[nu:])
            X[n] = gmres_cycle(sysm, Xold[n], b, k, precond)[0]
    return X, hist
