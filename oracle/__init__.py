"""CPU oracle for arXiv 2310.10430's inverted time-stepping iteration.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py
(cpu_baseline leg and ``--impl reference``) may import this package.  It
shares no code with the CUDA product in paper_2310_10430_b200/; the only
common module is workloads/ (seeded inputs, no arithmetic of the method).

Layout follows the paper: X = [U; P] with U[node*d + c].
The heavy loops (element integrals, CSR products, the iteration) are plain C
in biot_oracle.c; this file composes the global operators with scipy.sparse
(library primitives: COO->CSR summation and block stacking) exactly as
eqs. fullysystem / axb write them, restricts them to free DoFs
(reading R11), and converts to/from the node-interleaved vectors the
product's C-ABI exchanges (R20).

Pins: tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "biot_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.POINTER(ctypes.c_int64)
_i32 = ctypes.POINTER(ctypes.c_int32)


def build(force: bool = False) -> str:
    """Compile biot_oracle.c with gcc (-O2 -fopenmp).  Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_lame.argtypes = [ctypes.c_double, ctypes.c_double, _d, _d]
        L.oracle_beta.restype = ctypes.c_double
        L.oracle_beta.argtypes = [ctypes.c_double] * 3
        L.oracle_element.restype = ctypes.c_double
        L.oracle_element.argtypes = [ctypes.c_int, _d, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, _d, _d, _d, _d]
        L.oracle_assemble.restype = ctypes.c_int64
        L.oracle_assemble.argtypes = ([ctypes.c_int, ctypes.c_int64, _d, ctypes.c_int64, _i32,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double, _d]
                                      + [_i64, _i64, _d] * 2 + [_i64, _i64, _d, _d, _d])
        L.oracle_iterate.restype = ctypes.c_int
        L.oracle_iterate.argtypes = ([ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]
                                     + [_i64, _i32, _d] * 3
                                     + [ctypes.c_int32, _d, _d, _d, _d, ctypes.c_int32, ctypes.c_double, _d, _d,
                                        ctypes.c_int32])
        L.oracle_residual_norms.restype = ctypes.c_int
        L.oracle_residual_norms.argtypes = ([ctypes.c_int64, ctypes.c_int64, ctypes.c_int32]
                                            + [_i64, _i32, _d] * 2
                                            + [ctypes.c_int32, _d, _d, _d, _d, _d, ctypes.c_int32])
        _lib = L
    return _lib


def _p(a, t=_d):
    return a.ctypes.data_as(t)


def lame(E: float, nu: float):
    """P:L66-69."""
    lam, mu = ctypes.c_double(), ctypes.c_double()
    lib().oracle_lame(E, nu, ctypes.byref(lam), ctypes.byref(mu))
    return lam.value, mu.value


def beta(h: float, lam: float, mu: float) -> float:
    """P:L128-132."""
    return lib().oracle_beta(h, lam, mu)


def element(d: int, X: np.ndarray, lam: float, mu: float, alpha: float):
    """Element matrices (Ae, Be, Le, Me, |T|) of one simplex; see biot_oracle.c."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    nv = d + 1
    Ae = np.zeros((d * nv, d * nv)); Be = np.zeros((d * nv, nv))
    Le = np.zeros((nv, nv)); Me = np.zeros((nv, nv))
    vol = lib().oracle_element(d, _p(X), lam, mu, alpha, _p(Ae), _p(Be), _p(Le), _p(Me))
    return Ae, Be, Le, Me, vol


def _csr(m):
    m = sp.csr_matrix(m)
    m.sum_duplicates()
    m.sort_indices()
    return (np.ascontiguousarray(m.indptr, dtype=np.int64),
            np.ascontiguousarray(m.indices, dtype=np.int32),
            np.ascontiguousarray(m.data, dtype=np.float64))


@dataclass
class Blocks:
    A: sp.csr_matrix   # nu x nu  a(u,v) incl. lambda term (R7)
    B: sp.csr_matrix   # nu x np  -b(v,p)
    L: sp.csr_matrix   # np x np  int grad p . grad q
    C: sp.csr_matrix   # np x np  int kappa grad p . grad q (R9)
    M: sp.csr_matrix   # np x np  P1 mass (R8)


def assemble_blocks(dim, coords, cells, lam, mu, alpha, kappa) -> Blocks:
    """Global A, B, L, C, M (no boundary conditions) via the C element loop."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    cells = np.ascontiguousarray(cells, dtype=np.int32)
    kappa = np.ascontiguousarray(np.broadcast_to(kappa, (cells.shape[0],)), dtype=np.float64)
    nn, nc, d = coords.shape[0], cells.shape[0], dim
    nv = d + 1
    na, nb, npp = nc * (d * nv) ** 2, nc * d * nv * nv, nc * nv * nv
    Ai = np.empty(na, np.int64); Aj = np.empty(na, np.int64); Av = np.empty(na)
    Bi = np.empty(nb, np.int64); Bj = np.empty(nb, np.int64); Bv = np.empty(nb)
    Pi = np.empty(npp, np.int64); Pj = np.empty(npp, np.int64)
    Lv = np.empty(npp); Cv = np.empty(npp); Mv = np.empty(npp)
    bad = lib().oracle_assemble(d, nn, _p(coords), nc, _p(cells, _i32), lam, mu, alpha, _p(kappa),
                                _p(Ai, _i64), _p(Aj, _i64), _p(Av), _p(Bi, _i64), _p(Bj, _i64), _p(Bv),
                                _p(Pi, _i64), _p(Pj, _i64), _p(Lv), _p(Cv), _p(Mv))
    if bad:
        raise ValueError(f"degenerate or inverted cell {bad - 1}")
    nu = d * nn
    A = sp.coo_matrix((Av, (Ai, Aj)), shape=(nu, nu)).tocsr()
    B = sp.coo_matrix((Bv, (Bi, Bj)), shape=(nu, nn)).tocsr()
    L = sp.coo_matrix((Lv, (Pi, Pj)), shape=(nn, nn)).tocsr()
    C = sp.coo_matrix((Cv, (Pi, Pj)), shape=(nn, nn)).tocsr()
    M = sp.coo_matrix((Mv, (Pi, Pj)), shape=(nn, nn)).tocsr()
    for m in (A, B, L, C, M):
        m.sum_duplicates(); m.sort_indices()
    return Blocks(A, B, L, C, M)


def traction_load(dim, coords, facets, traction) -> np.ndarray:
    """F_u = int_{Gamma_N} t . phi ds for constant t (P:L223-227 'F^m'; R16).

    Exact for P1: int_f phi_a ds = |f| / d for each of the d vertices of a
    boundary facet f (|f| = edge length in 2D, triangle area in 3D).
    Returns F_u (node-major, length d*N).
    """
    nn = coords.shape[0]
    F = np.zeros(dim * nn)
    for f in np.asarray(facets):
        P = coords[f]
        if dim == 2:
            meas = float(np.linalg.norm(P[1] - P[0]))
        else:
            meas = 0.5 * float(np.linalg.norm(np.cross(P[1] - P[0], P[2] - P[0])))
        for a in f:
            for c in range(dim):
                F[a * dim + c] += meas / dim * traction[c]
    return F


# Quadrature of the source loads (reading R24): barycentric points, weights relative to
# the cell measure.  Triangles: the symmetric 7-point rule exact for degree 5
# (Strang & Fix / Dunavant); tetrahedra: the symmetric 4-point degree-2 rule.
_TRI7_A1, _TRI7_B1 = 0.059715871789770, 0.470142064105115
_TRI7_A2, _TRI7_B2 = 0.797426985353087, 0.101286507323456
_QUAD = {
    2: (np.array([[1 / 3, 1 / 3, 1 / 3],
                  [_TRI7_A1, _TRI7_B1, _TRI7_B1], [_TRI7_B1, _TRI7_A1, _TRI7_B1], [_TRI7_B1, _TRI7_B1, _TRI7_A1],
                  [_TRI7_A2, _TRI7_B2, _TRI7_B2], [_TRI7_B2, _TRI7_A2, _TRI7_B2], [_TRI7_B2, _TRI7_B2, _TRI7_A2]]),
        np.array([0.225] + [0.132394152788506] * 3 + [0.125939180544827] * 3)),
    3: (np.array([[0.5854101966249685] + [0.1381966011250105] * 3,
                  [0.1381966011250105, 0.5854101966249685, 0.1381966011250105, 0.1381966011250105],
                  [0.1381966011250105, 0.1381966011250105, 0.5854101966249685, 0.1381966011250105],
                  [0.1381966011250105] * 3 + [0.5854101966249685]]),
        np.full(4, 0.25)),
}


def source_load(dim, coords, cells, fn, q, dt):
    """[int f_q . phi_a ; -dt int g_q phi_a] (f^m = [F^m; -tau G^m], G^m = (g, q_h))
    for source field q of fn (fn(q, xyz) -> [npts, dim+1]) by the quadrature _QUAD.
    Returns paper order [U (node-major); P]."""
    lam, w = _QUAD[dim]
    X = coords[cells]                                     # (nc, d+1, d)
    E = X[:, 1:, :] - X[:, :1, :]                         # edge matrix rows
    vol = np.abs(np.linalg.det(E)) / (2.0 if dim == 2 else 6.0)
    xq = np.einsum("ka,cad->ckd", lam, X)                 # (nc, nq, d)
    vals = np.asarray(fn(q, xq.reshape(-1, dim)), dtype=np.float64).reshape(cells.shape[0], len(w), dim + 1)
    # contribution of cell c to its vertex a: |T| sum_k w_k lam_k[a] v(x_k)
    contrib = np.einsum("c,k,ka,ckv->cav", vol, w, lam, vals)   # (nc, d+1, d+1 comps)
    nn = coords.shape[0]
    out = np.zeros((nn, dim + 1))
    np.add.at(out, cells.reshape(-1), contrib.reshape(-1, dim + 1))
    return np.concatenate([out[:, :dim].reshape(-1), -dt * out[:, dim]])


class OracleSystem:
    """The per-step operators AA, A' and load f of one problem (free DoFs only).

    Built from a workloads.Problem-like object (fields dim, coords, cells,
    lam, mu, alpha, storage, kappa, h, dt, dirichlet, facets, traction; optional
    sources / source_coef / dirichlet_values / dirichlet_coef of §4.1).
    `beta_override` replaces the printed beta formula (R5).

    Load of step n ("f^m"): f^n = sum_j coef_j(n) loads[j] with
    loads[0] = F (traction, coefficient s_n, R16) and, for §4.1 problems (R24),
    one term [(f_q, phi); -tau (g_q, phi)] per source field q (source_load) with
    coefficient source_coef[q][n-1], then the Dirichlet lifting -AA_{free,D} x_D
    (coefficient c_n) and A'_{free,D} x_D (coefficient c_{n-1}), x_D(t_n) = c_n x_D.
    """

    def __init__(self, prob, dt=None, beta_override=None, dirichlet=None):
        d = prob.dim
        self.dim = d
        self.nn = prob.coords.shape[0]
        self.nu = d * self.nn
        self.np = self.nn
        self.ndof = self.nu + self.np
        self.dt = prob.dt if dt is None else dt
        self.blocks = bl = assemble_blocks(d, prob.coords, prob.cells, prob.lam, prob.mu,
                                           prob.alpha, prob.kappa)
        self.beta = beta(prob.h, prob.lam, prob.mu) if beta_override is None else beta_override
        S, tau, b = prob.storage, self.dt, self.beta
        # S~p = S M + tau C + beta L (P:L259-262 with R8, R9);  H = S M + beta L (A' block)
        self.St = (S * bl.M + tau * bl.C + b * bl.L).tocsr()
        self.H = (S * bl.M + b * bl.L).tocsr()
        AA = sp.bmat([[bl.A, bl.B], [bl.B.T, -self.St]], format="csr")
        AP = sp.bmat([[sp.csr_matrix((self.nu, self.nu)), sp.csr_matrix((self.nu, self.np))],
                      [bl.B.T, -self.H]], format="csr")
        mask = prob.dirichlet if dirichlet is None else dirichlet
        m = np.asarray(mask, dtype=np.uint8).reshape(self.nn, d + 1)
        self.free = np.concatenate([(m[:, :d] == 0).ravel(), m[:, d] == 0]).astype(np.float64)
        Df = sp.diags(self.free)
        self.AA = (Df @ AA @ Df).tocsr(); self.AA.eliminate_zeros()
        self.AP = (Df @ AP @ Df).tocsr(); self.AP.eliminate_zeros()
        Fu = traction_load(d, prob.coords, prob.facets, prob.traction)
        self.F = np.concatenate([Fu, np.zeros(self.np)]) * self.free
        # further load terms of §4.1 (R24); kinds: ("src", q), ("dnow",), ("dprev",)
        self.loads = [self.F]
        self.kinds = [("scale",)]
        self.prob = prob
        fn = getattr(prob, "source_fn", None)
        if fn is not None:
            for q in range(int(prob.n_sources)):
                self.loads.append(source_load(d, np.asarray(prob.coords, dtype=np.float64),
                                              np.asarray(prob.cells), fn, q, self.dt) * self.free)
                self.kinds.append(("src", q))
        dv = getattr(prob, "dirichlet_values", None)
        if dv is not None:
            xD = self.to_paper(np.asarray(dv, dtype=np.float64)) * (1.0 - self.free)
            self.loads.append(-(AA @ xD) * self.free)
            self.kinds.append(("dnow",))
            self.loads.append((AP @ xD) * self.free)
            self.kinds.append(("dprev",))
        self.Fall = np.ascontiguousarray(np.array(self.loads))
        fu, fp = self.free[:self.nu], self.free[self.nu:]
        self.BT = (sp.diags(fp) @ bl.B.T.tocsr() @ sp.diags(fu)).tocsr(); self.BT.eliminate_zeros()
        dA = bl.A.diagonal()
        dS = self.St.diagonal()
        self.DAinv = np.where(fu > 0, 1.0 / np.where(fu > 0, dA, 1.0), 0.0)
        self.DSinv = np.where(fp > 0, 1.0 / np.where(fp > 0, dS, 1.0), 0.0)
        self._AA = _csr(self.AA); self._AP = _csr(self.AP); self._BT = _csr(self.BT)

    # -- layout conversions (R20) -------------------------------------------------
    def to_paper(self, x):
        """node-interleaved [..., N*(d+1)] -> paper order [..., d*N + N]."""
        x = np.asarray(x, dtype=np.float64)
        d, nn = self.dim, self.nn
        xr = x.reshape(x.shape[:-1] + (nn, d + 1))
        U = xr[..., :d].reshape(x.shape[:-1] + (d * nn,))
        return np.concatenate([U, xr[..., d]], axis=-1)

    def from_paper(self, X):
        X = np.asarray(X, dtype=np.float64)
        d, nn = self.dim, self.nn
        out = np.empty(X.shape[:-1] + (nn, d + 1))
        out[..., :d] = X[..., :d * nn].reshape(X.shape[:-1] + (nn, d))
        out[..., d] = X[..., d * nn:]
        return out.reshape(X.shape[:-1] + (nn * (d + 1),))

    # -- loads -------------------------------------------------------------------
    def coefs(self, s, first_step=1, nt=None):
        """[J, nt] coefficients of the load terms for global steps first_step..: row 0 is
        the traction scale s (length nt, the window's own), the rest from the problem."""
        s = np.asarray(s, dtype=np.float64)
        nt = s.shape[-1] if nt is None else nt
        C = np.zeros((len(self.loads), nt))
        C[0] = s
        n = np.arange(first_step, first_step + nt)
        for j, k in enumerate(self.kinds):
            if k[0] == "src":
                C[j] = np.asarray(self.prob.source_coef)[k[1]][n - 1]
            elif k[0] == "dnow":
                dc = getattr(self.prob, "dirichlet_coef", None)
                C[j] = 1.0 if dc is None else np.asarray(dc)[n]
            elif k[0] == "dprev":
                dc = getattr(self.prob, "dirichlet_coef", None)
                C[j] = 1.0 if dc is None else np.asarray(dc)[n - 1]
        return C

    def _loadset(self, s):
        S = np.ascontiguousarray(np.atleast_2d(np.asarray(s, dtype=np.float64)))
        Fm = self.F[None] if S.shape[0] == 1 else self.Fall
        assert S.shape[0] == Fm.shape[0], "coefficient rows must match the load terms"
        return S, np.ascontiguousarray(Fm)

    def load_vec(self, s, n):
        """f^n = sum_j S[j, n-1] loads[j] for s of shape (nt,) (traction only) or (J, nt)."""
        S, Fm = self._loadset(s)
        return S[:, n - 1] @ Fm

    # -- the iteration ------------------------------------------------------------
    def iterate(self, X, s, K, precond=2, omega=0.5, history=True, nthreads=0):
        """K Jacobi-in-time outer iterations in place on X[(nt+1), ndof] (paper order).

        X[0] is the fixed previous state (x_0 or a window's ghost).  Returns the
        residual-norm history [K, nt, 2] (norms of r at x^k, k = 0..K-1) or None.
        """
        X = np.ascontiguousarray(X, dtype=np.float64)
        nt = X.shape[0] - 1
        S, Fm = self._loadset(s)
        assert S.shape[1] == nt and X.shape[1] == self.ndof and precond in (1, 2)
        hist = np.zeros((max(K, 1), nt, 2)) if history else None
        rc = lib().oracle_iterate(self.nu, self.np, nt, K,
                                  _p(self._AA[0], _i64), _p(self._AA[1], _i32), _p(self._AA[2]),
                                  _p(self._AP[0], _i64), _p(self._AP[1], _i32), _p(self._AP[2]),
                                  _p(self._BT[0], _i64), _p(self._BT[1], _i32), _p(self._BT[2]),
                                  S.shape[0], _p(Fm), _p(S), _p(self.DAinv), _p(self.DSinv),
                                  precond, omega, _p(X), _p(hist) if history else None, nthreads)
        if rc != 0:
            raise MemoryError("oracle_iterate failed")
        return X, (hist[:K] if history else None)

    def residual_norms(self, X, s, nthreads=0, return_r=False):
        """||r_{n,u}||, ||r_{n,p}|| at X without updating (R12); [nt, 2]."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        nt = X.shape[0] - 1
        S, Fm = self._loadset(s)
        assert S.shape[1] == nt
        out = np.zeros((nt, 2))
        r = np.zeros((nt, self.ndof)) if return_r else None
        rc = lib().oracle_residual_norms(self.nu, self.np, nt,
                                         _p(self._AA[0], _i64), _p(self._AA[1], _i32), _p(self._AA[2]),
                                         _p(self._AP[0], _i64), _p(self._AP[1], _i32), _p(self._AP[2]),
                                         S.shape[0], _p(Fm), _p(S), _p(X), _p(out),
                                         _p(r) if return_r else None, nthreads)
        if rc != 0:
            raise MemoryError("oracle_residual_norms failed")
        return (out, r) if return_r else out


def run(prob, x0_steps, s, K, precond=2, omega=0.5, ghost=None, nthreads=0, history=True):
    """Convenience: node-interleaved in/out.

    x0_steps: [nt, ndof] initial iterates x_n^0 for the window's steps;
    ghost: x of the step before the window (default: zero initial state).
    Returns (x^K [nt, ndof] node-interleaved, history [K, nt, 2], system).
    """
    sysm = prob if isinstance(prob, OracleSystem) else OracleSystem(prob)
    nt = x0_steps.shape[0]
    X = np.zeros((nt + 1, sysm.ndof))
    if ghost is not None:
        X[0] = sysm.to_paper(ghost)
    X[1:] = sysm.to_paper(x0_steps)
    X, hist = sysm.iterate(X, s, K, precond, omega, history=history, nthreads=nthreads)
    return sysm.from_paper(X[1:]), hist, sysm
