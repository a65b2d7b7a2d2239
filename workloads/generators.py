"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no element integrals, no
operators, no preconditioner, no iteration).  It only produces the *inputs*
that the paper's problem statement takes (§2.1; L523, §4.1
"uniform mesh"), shaped like BASELINE.json's five configs:

* structured simplicial meshes of the unit square / cube (node coordinates
  and cell connectivity),
* the Dirichlet node sets of the Terzaghi-type column (which DoFs are fixed),
* the boundary facets that carry the top traction and the traction vector,
* per-cell permeability kappa (uniform or lognormal, counter-based RNG),
* the seeded initial iterate x^0 and the load scales s_n.

Both the oracle and the CUDA library receive identical arrays from here and
each computes everything else independently.

Counter-based generator (reading R18): SplitMix64 finaliser
``sm64``; the k-th uniform of stream ``seed`` is
``u_k = ((sm64(sm64(seed) + k) >> 11) + 0.5) * 2**-53`` and a standard normal
is Box-Muller ``z_e = sqrt(-2 ln u_{2e}) cos(2 pi u_{2e+1})``.  Every value
depends only on (seed, index), never on generation order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def sm64(x):
    """SplitMix64 finaliser on uint64 numpy arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, k: np.ndarray) -> np.ndarray:
    """k-th uniform in (0,1) of stream `seed` (k: uint64 array)."""
    base = sm64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    with np.errstate(over="ignore"):
        bits = sm64(base + np.asarray(k, dtype=np.uint64))
    return ((bits >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def std_normal(seed: int, idx: np.ndarray) -> np.ndarray:
    """Standard normal z_idx of stream `seed` (Box-Muller on u_{2i}, u_{2i+1})."""
    idx = np.asarray(idx, dtype=np.uint64)
    u1 = uniform01(seed, idx * np.uint64(2))
    u2 = uniform01(seed, idx * np.uint64(2) + np.uint64(1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


# --------------------------------------------------------------------------
# meshes (uniform structured mesh, h = 1/2^k; 3D per BJ cfg 4-5)
# --------------------------------------------------------------------------

def mesh_square(n: int):
    """Unit square, n x n cells, each split by the BL->TR diagonal.

    node id = j*(n+1) + i at (i/n, j/n); cell (i,j) -> triangles
    (n00, n10, n11) and (n00, n11, n01), counter-clockwise.
    Returns coords (N,2) float64, cells (2n^2, 3) int32.
    """
    w = n + 1
    ii, jj = np.meshgrid(np.arange(w), np.arange(w), indexing="xy")
    coords = np.stack([ii.ravel() / n, jj.ravel() / n], axis=1).astype(np.float64)
    ci, cj = np.meshgrid(np.arange(n), np.arange(n), indexing="xy")
    n00 = (cj * w + ci).ravel()
    n10 = n00 + 1
    n11 = n00 + w + 1
    n01 = n00 + w
    cells = np.empty((2 * n * n, 3), dtype=np.int32)
    cells[0::2] = np.stack([n00, n10, n11], axis=1)
    cells[1::2] = np.stack([n00, n11, n01], axis=1)
    return coords, cells


_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def mesh_cube(n: int):
    """Unit cube, n^3 cells, each split into 6 Kuhn tetrahedra.

    node id = (k*(n+1) + j)*(n+1) + i at (i,j,k)/n.  For each permutation
    (a,b,c) of the axes the tet is {v, v+e_a, v+e_a+e_b, v+e_a+e_b+e_c};
    vertices are reordered (swap of the last two) so that every tet is
    positively oriented.  Returns coords (N,3), cells (6n^3, 4) int32.
    """
    w = n + 1
    kk, jj, ii = np.meshgrid(np.arange(w), np.arange(w), np.arange(w), indexing="ij")
    coords = np.stack([ii.ravel() / n, jj.ravel() / n, kk.ravel() / n], axis=1).astype(np.float64)
    stride = np.array([1, w, w * w], dtype=np.int64)
    ck, cj, ci = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    v = (ck * w * w + cj * w + ci).ravel().astype(np.int64)
    cells = np.empty((6 * n ** 3, 4), dtype=np.int32)
    for p, (a, b, c) in enumerate(_PERMS):
        e = np.eye(3, dtype=np.int64)
        o1 = e[a]
        o2 = e[a] + e[b]
        tet_off = [0, int(o1 @ stride), int(o2 @ stride), int(stride.sum())]
        # orientation of the offset simplex (same for every cube)
        m = np.stack([o1, o2, np.ones(3, dtype=np.int64)], axis=0)
        det = int(round(np.linalg.det(m.astype(np.float64))))
        if det < 0:
            tet_off[2], tet_off[3] = tet_off[3], tet_off[2]
        cells[p::6] = np.stack([v + t for t in tet_off], axis=1)
    return coords, cells


def mesh(dim: int, n: int):
    return mesh_square(n) if dim == 2 else mesh_cube(n)


# --------------------------------------------------------------------------
# boundary description of the Terzaghi-type column (BJ configs)
# --------------------------------------------------------------------------

def column_dirichlet(coords: np.ndarray) -> np.ndarray:
    """Node-interleaved Dirichlet mask [u_1..u_d, p] per node (uint8).

    2D: u_x=0 on x in {0,1}; u=0 on y=0; p=0 on y=1.
    3D: u_x=0 on x in {0,1}; u_y=0 on y in {0,1}; u=0 on z=0; p=0 on z=1.
    (BJ configs: drained top, roller sides, fixed bottom.)
    """
    nn, d = coords.shape
    eps = 1e-12
    mask = np.zeros((nn, d + 1), dtype=np.uint8)
    for ax in range(d - 1):
        side = (coords[:, ax] < eps) | (coords[:, ax] > 1 - eps)
        mask[side, ax] = 1
    bottom = coords[:, d - 1] < eps
    top = coords[:, d - 1] > 1 - eps
    mask[bottom, :d] = 1
    mask[top, d] = 1
    return mask.reshape(-1)


def top_facets(coords: np.ndarray, cells: np.ndarray) -> np.ndarray:
    """Boundary facets lying on the top face (y=1 in 2D, z=1 in 3D).

    A facet is d vertices of one cell that all lie on the top face; the
    result is (n_facets, d) int32.  Selection only, no integration.
    """
    d = coords.shape[1]
    on_top = coords[:, d - 1] > 1 - 1e-12
    flags = on_top[cells]                      # (nc, d+1)
    sel = flags.sum(axis=1) == d
    c = cells[sel]
    f = flags[sel]
    out = c[f].reshape(-1, d)
    return out.astype(np.int32)


def kappa_cells(n_cells: int, median: float, sigma: float = 0.0, seed: int = 0) -> np.ndarray:
    """Per-cell permeability: uniform `median`, or lognormal median*exp(sigma z_e)."""
    if sigma == 0.0:
        return np.full(n_cells, median, dtype=np.float64)
    z = std_normal(seed, np.arange(n_cells, dtype=np.uint64))
    return median * np.exp(sigma * z)


def initial_iterate(dirichlet: np.ndarray, n_steps: np.ndarray, seed: int) -> np.ndarray:
    """Seeded x_n^0 ~ N(0,1) on free DoFs, 0 on Dirichlet DoFs.

    `n_steps` are global step indices n (1-based); row r of the result is
    x_{n_steps[r]}^0, node-interleaved.  Value at (n, dof) is
    z(seed, (n-1)*N_dof + dof), independent of which steps are requested.
    """
    ndof = dirichlet.size
    n_steps = np.asarray(n_steps, dtype=np.int64)
    out = np.empty((n_steps.size, ndof), dtype=np.float64)
    free = dirichlet == 0
    base = np.arange(ndof, dtype=np.uint64)
    for r, n in enumerate(n_steps):
        z = std_normal(seed, np.uint64((int(n) - 1) * ndof) + base)
        out[r] = np.where(free, z, 0.0)
    return out


def load_scales(n_t: int, parity: bool) -> np.ndarray:
    """s_n for n=1..N_t: 1 (metric runs, BJ 'unit load') or 1+0.1 sin n (parity)."""
    n = np.arange(1, n_t + 1, dtype=np.float64)
    return 1.0 + 0.1 * np.sin(n) if parity else np.ones(n_t)


# --------------------------------------------------------------------------
# problem bundle
# --------------------------------------------------------------------------

# --------------------------------------------------------------------------
# manufactured-solution inputs (§4.1)
# --------------------------------------------------------------------------

def lame_from_young(E: float, nu: float):
    """Problem parameters E, nu -> (lambda, mu), the conversion P:L66-69 states."""
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def all_boundary_dirichlet(coords: np.ndarray) -> np.ndarray:
    """Every DoF of every boundary node fixed ("Dirichlet boundary conditions
    are used at all boundaries")."""
    nn, d = coords.shape
    eps = 1e-12
    on = np.zeros(nn, dtype=bool)
    for ax in range(d):
        on |= (coords[:, ax] < eps) | (coords[:, ax] > 1 - eps)
    mask = np.zeros((nn, d + 1), dtype=np.uint8)
    mask[on, :] = 1
    return mask.reshape(-1)


def trig_source(lam, mu, alpha, K):
    """§4.1's data as a function of position: source_fn(q, xyz) -> [npts, 3]
    node-interleaved (f_1, f_2, g); q = 0 the cos(t) parts, q = 1 the sin(t) part:

      f = -3 pi cos t (alpha s_x c_y - 3 pi (lam + 3 mu) c c + 3 pi (lam + mu) s s,
                       alpha c_x s_y - 3 pi (lam + 3 mu) c c + 3 pi (lam + mu) s s),
      g = 3 alpha pi sin t (c_x s_y + s_x c_y) + 18 K pi^2 cos t c c
    (c_x = cos 3 pi x, s_x = sin 3 pi x, ...).  The printed minus sign in g is a
    typo (reading R13): the stated exact solution needs the plus."""
    pi = math.pi

    def fn(q, xyz):
        x, y = xyz[:, 0], xyz[:, 1]
        cx, cy = np.cos(3 * pi * x), np.cos(3 * pi * y)
        sx, sy = np.sin(3 * pi * x), np.sin(3 * pi * y)
        cc, ss = cx * cy, sx * sy
        out = np.zeros((xyz.shape[0], 3))
        if q == 0:
            out[:, 0] = -3 * pi * (alpha * sx * cy - 3 * pi * (lam + 3 * mu) * cc + 3 * pi * (lam + mu) * ss)
            out[:, 1] = -3 * pi * (alpha * cx * sy - 3 * pi * (lam + 3 * mu) * cc + 3 * pi * (lam + mu) * ss)
            out[:, 2] = 18 * K * pi ** 2 * cc
        else:
            out[:, 2] = 3 * alpha * pi * (cx * sy + sx * cy)
        return out
    return fn


def trig_exact(xyz, t):
    """The exact solution of §4.1: p = u_1 = u_2 = cos t cos 3 pi x cos 3 pi y."""
    return math.cos(t) * np.cos(3 * math.pi * xyz[:, 0]) * np.cos(3 * math.pi * xyz[:, 1])


def trig_problem(k: int, n_t: int, dt: float, name: str = ""):
    """§4.1 trigonometric test: unit square, h = 2^-k, E = 1, nu = 0.3,
    alpha = 1, K = 1, Dirichlet data on all boundaries, no storage term.  Steps
    t_n = n dt, n = 1..n_t; sources with per-step coefficients (cos t_n, sin t_n),
    Dirichlet values x_D = cos 3 pi x cos 3 pi y (every component) with c_n = cos t_n,
    x_0 = the initial condition.
    """
    n = 2 ** k
    coords, cells = mesh_square(n)
    lam, mu = lame_from_young(1.0, 0.3)
    alpha, K = 1.0, 1.0
    prof = np.repeat(trig_exact(coords, 0.0), 3)
    t = np.arange(0, n_t + 1, dtype=np.float64) * dt
    p = Problem(dim=2, n=n, n_t=n_t, dt=dt, K=0, lam=lam, mu=mu, alpha=alpha, storage=0.0,
                kappa=np.full(cells.shape[0], K), h=1.0 / n, coords=coords, cells=cells,
                dirichlet=all_boundary_dirichlet(coords), facets=np.zeros((0, 2), np.int32),
                traction=np.zeros(2), x0_seed=0, name=name or f"trig_h{n}")
    p.source_fn = trig_source(lam, mu, alpha, K)
    p.n_sources = 2
    p.source_coef = np.stack([np.cos(t[1:]), np.sin(t[1:])])
    p.dirichlet_values = prof
    p.dirichlet_coef = np.cos(t)
    p.x_initial = prof.copy()
    p.meta = dict(E=1.0, nu=0.3, K=K)
    return p


_PATCH = dict(A=(0.3, -0.7, 0.2), B=(-0.1, 0.4, 0.9), C=(0.5, 1.3, -0.6))


def patch_exact(xyz, t):
    """Exact solution of linear_patch_problem at time t, node-interleaved [u_1, u_2, p]."""
    A, B, C = _PATCH["A"], _PATCH["B"], _PATCH["C"]
    x, y = xyz[:, 0], xyz[:, 1]
    prof = np.stack([A[0] + A[1] * x + A[2] * y, B[0] + B[1] * x + B[2] * y,
                     C[0] + C[1] * x + C[2] * y], axis=1)
    return ((1.0 + t) * prof).reshape(-1)


def linear_patch_problem(n: int, n_t: int, dt: float, lam=1.0, mu=1.0, alpha=1.0, K=1.0):
    """A manufactured solution that P1-P1 backward Euler reproduces exactly (test input):
    u_1 = (1+t) a(x), u_2 = (1+t) b(x), p = (1+t) c(x) with a, b, c affine.  Then
    -div sigma = 0, f = alpha grad p = (1+t) alpha grad c (constant in space),
    g = alpha div u_t - K lap p = alpha div (a, b) (constant); all boundaries Dirichlet.
    Sources: q = 0 the f-part (coefficient 1 + t_n), q = 1 the g-part (coefficient 1)."""
    coords, cells = mesh_square(n)
    A, B, C = _PATCH["A"], _PATCH["B"], _PATCH["C"]

    def fn(q, xyz):
        out = np.zeros((xyz.shape[0], 3))
        if q == 0:
            out[:, 0] = alpha * C[1]
            out[:, 1] = alpha * C[2]
        else:
            out[:, 2] = alpha * (A[1] + B[2])
        return out
    t = np.arange(0, n_t + 1, dtype=np.float64) * dt
    p = Problem(dim=2, n=n, n_t=n_t, dt=dt, K=0, lam=lam, mu=mu, alpha=alpha, storage=0.0,
                kappa=np.full(cells.shape[0], K), h=1.0 / n, coords=coords, cells=cells,
                dirichlet=all_boundary_dirichlet(coords), facets=np.zeros((0, 2), np.int32),
                traction=np.zeros(2), x0_seed=0, name=f"patch_h{n}")
    p.source_fn = fn
    p.n_sources = 2
    p.source_coef = np.stack([1.0 + t[1:], np.ones(n_t)])
    p.dirichlet_values = patch_exact(coords, 0.0)
    p.dirichlet_coef = 1.0 + t
    p.x_initial = p.dirichlet_values.copy()
    return p


@dataclass
class Problem:
    dim: int
    n: int                     # cells per axis
    n_t: int
    dt: float
    K: int
    lam: float
    mu: float
    alpha: float
    storage: float
    kappa: np.ndarray          # per cell
    h: float
    coords: np.ndarray
    cells: np.ndarray
    dirichlet: np.ndarray      # node-interleaved uint8
    facets: np.ndarray         # (nf, d) int32
    traction: np.ndarray       # (d,)
    x0_seed: int
    name: str = ""
    meta: dict = field(default_factory=dict)
    # §4.1 data (optional): source_fn(q, xyz [npts, d]) -> [npts, d+1] for q < n_sources
    # with [n_sources][n_t] coefficients; Dirichlet values x_D with coefficients
    # c_0..c_{n_t}; x_0
    source_fn: object = None
    n_sources: int = 0
    source_coef: np.ndarray = None
    dirichlet_values: np.ndarray = None
    dirichlet_coef: np.ndarray = None
    x_initial: np.ndarray = None

    @property
    def n_nodes(self) -> int:
        return self.coords.shape[0]

    @property
    def n_dof(self) -> int:
        return self.coords.shape[0] * (self.dim + 1)


def make_problem(dim, n, n_t, dt, K, lam=1.0, mu=1.0, alpha=1.0, storage=1e-3,
                 kappa_median=1e-2, kappa_sigma=0.0, kappa_seed=0, x0_seed=0, name=""):
    coords, cells = mesh(dim, n)
    kap = kappa_cells(cells.shape[0], kappa_median, kappa_sigma, kappa_seed)
    dirichlet = column_dirichlet(coords)
    facets = top_facets(coords, cells)
    traction = np.zeros(dim)
    traction[dim - 1] = -1.0
    return Problem(dim=dim, n=n, n_t=n_t, dt=dt, K=K, lam=lam, mu=mu, alpha=alpha,
                   storage=storage, kappa=kap, h=1.0 / n, coords=coords, cells=cells,
                   dirichlet=dirichlet, facets=facets, traction=traction,
                   x0_seed=x0_seed, name=name)
