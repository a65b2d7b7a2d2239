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
