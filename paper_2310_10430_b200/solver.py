"""Thin Python front end of the C-ABI (same names as include/biot_pit.h).

    s = BiotSolver(problem, n_t, dt, precond=2, omega=0.5)
    s.set_iterate(1, x0)            # optional seeded x_n^0
    s.iterate(K)                    # biot_iterate
    s.residual_norms()              # biot_residual_norms -> [n_t_local, 2]
    s.solution(n, count)            # biot_solution -> [count, n_dof]

Argument marshalling only; all work runs in libbiot_pit.so.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import BiotOpts, BiotInfo, Inputs, check, ptr


def assemble_host(prob, dt, beta=None):
    """biot_assemble_host: the library's assembled AA, A' (COO, node-interleaved), f, dinv."""
    L = _lib.load()
    inp = Inputs(prob, beta=beta)
    na, npp = ctypes.c_int64(), ctypes.c_int64()
    z = ctypes.POINTER(ctypes.c_int64)()
    zd = ctypes.POINTER(ctypes.c_double)()
    check(L.biot_assemble_host(ctypes.byref(inp.mesh), ctypes.byref(inp.mat), ctypes.byref(inp.bc), dt,
                               ctypes.byref(na), z, z, zd, ctypes.byref(npp), z, z, zd, zd, zd))
    ndof = prob.coords.shape[0] * (prob.dim + 1)
    Ai = np.empty(na.value, np.int64); Aj = np.empty(na.value, np.int64); Av = np.empty(na.value)
    Pi = np.empty(npp.value, np.int64); Pj = np.empty(npp.value, np.int64); Pv = np.empty(npp.value)
    f = np.empty(ndof); dinv = np.empty(ndof)
    I64 = ctypes.POINTER(ctypes.c_int64)
    check(L.biot_assemble_host(ctypes.byref(inp.mesh), ctypes.byref(inp.mat), ctypes.byref(inp.bc), dt,
                               ctypes.byref(na), ptr(Ai, I64), ptr(Aj, I64), ptr(Av),
                               ctypes.byref(npp), ptr(Pi, I64), ptr(Pj, I64), ptr(Pv), ptr(f), ptr(dinv)))
    return (Ai, Aj, Av), (Pi, Pj, Pv), f, dinv


def mesh_structured(dim, n):
    """biot_mesh_structured: (coords [N, dim], cells [nc, dim+1]) of the library's
    structured unit square / Kuhn cube (copied out, library buffers released)."""
    L = _lib.load()
    X = ctypes.POINTER(ctypes.c_double)()
    C = ctypes.POINTER(ctypes.c_int32)()
    nn, nc = ctypes.c_int64(), ctypes.c_int64()
    check(L.biot_mesh_structured(dim, n, ctypes.byref(X), ctypes.byref(C), ctypes.byref(nn), ctypes.byref(nc)))
    try:
        coords = np.ctypeslib.as_array(X, shape=(nn.value, dim)).copy()
        cells = np.ctypeslib.as_array(C, shape=(nc.value, dim + 1)).copy()
    finally:
        L.biot_free(ctypes.cast(X, ctypes.c_void_p))
        L.biot_free(ctypes.cast(C, ctypes.c_void_p))
    return coords, cells


def bc_column(coords, cells, load=1.0):
    """biot_bc_column: (dirichlet mask, load vector F, top facets) of the column problem."""
    from ._lib import BiotMesh
    L = _lib.load()
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    cells = np.ascontiguousarray(cells, dtype=np.int32)
    dim = coords.shape[1]
    mesh = BiotMesh(dim, coords.shape[0], ptr(coords), cells.shape[0], ptr(cells, ctypes.POINTER(ctypes.c_int32)))
    nf = ctypes.c_int64()
    check(L.biot_bc_column(ctypes.byref(mesh), load, None, None, ctypes.byref(nf), None))
    mask = np.zeros(coords.shape[0] * (dim + 1), np.uint8)
    F = np.zeros(coords.shape[0] * (dim + 1))
    facets = np.zeros((nf.value, dim), np.int32)
    check(L.biot_bc_column(ctypes.byref(mesh), load, ptr(mask, ctypes.POINTER(ctypes.c_uint8)), ptr(F),
                           ctypes.byref(nf), ptr(facets, ctypes.POINTER(ctypes.c_int32))))
    return mask, F, facets


def assemble_loads_host(prob, dt, beta=None):
    """biot_assemble_loads_host: the library's further load terms (R24), node-interleaved
    [n_terms, n_dof], with their kinds (0 source, 1 lifting at c_n, 2 at c_{n-1}) and
    source indices."""
    L = _lib.load()
    inp = Inputs(prob, beta=beta)
    n = ctypes.c_int32()
    I32 = ctypes.POINTER(ctypes.c_int32)
    check(L.biot_assemble_loads_host(ctypes.byref(inp.mesh), ctypes.byref(inp.mat), ctypes.byref(inp.bc), dt,
                                     ctypes.byref(n), None, None, None))
    ndof = prob.coords.shape[0] * (prob.dim + 1)
    F = np.zeros((n.value, ndof))
    kinds = np.zeros(n.value, np.int32)
    src = np.zeros(n.value, np.int32)
    check(L.biot_assemble_loads_host(ctypes.byref(inp.mesh), ctypes.byref(inp.mat), ctypes.byref(inp.bc), dt,
                                     ctypes.byref(n), ptr(F), ptr(kinds, I32), ptr(src, I32)))
    if inp.cb_error is not None:
        raise inp.cb_error
    return F, kinds, src


class BiotSolver:
    def __init__(self, prob, n_t=None, dt=None, precond=2, omega=0.5, device=0, rank=0, world=1,
                 nccl_id=None, stream=None, flags=0, history=0, load_scale=None, x_initial=None,
                 beta=None):
        self.lib = _lib.load()
        self.prob = prob
        self.n_t = prob.n_t if n_t is None else n_t
        self.dt = prob.dt if dt is None else dt
        self._inp = Inputs(prob, load_scale=load_scale, x_initial=x_initial, beta=beta)
        self._nccl_id = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), 128)
        opts = BiotOpts(precond, omega, device, rank, world,
                        ctypes.cast(self._nccl_id, ctypes.c_void_p) if self._nccl_id is not None else None,
                        stream, flags, history)
        self.ctx = ctypes.c_void_p()
        check(self.lib.biot_setup(ctypes.byref(self._inp.mesh), ctypes.byref(self._inp.mat),
                                  ctypes.byref(self._inp.bc), self.dt, self.n_t, ctypes.byref(opts),
                                  ctypes.byref(self.ctx)))
        self.info = self.get_info()
        self.ndof = self.info.n_dof
        self.n_tl = self.info.n_t_local
        self.first_step = self.info.first_step

    # --- ABI calls ---------------------------------------------------------------
    def get_info(self):
        inf = BiotInfo()
        check(self.lib.biot_get_info(self.ctx, ctypes.byref(inf)), self.ctx)
        return inf

    def set_iterate(self, n, x):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, self.ndof)
        check(self.lib.biot_set_iterate(self.ctx, n, x.shape[0], ptr(x)), self.ctx)

    def set_load_scale(self, s):
        s = np.ascontiguousarray(s, dtype=np.float64)
        assert s.shape == (self.n_t,)
        check(self.lib.biot_set_load_scale(self.ctx, ptr(s)), self.ctx)

    def iterate_gs(self, K):
        check(self.lib.biot_iterate_gs(self.ctx, K), self.ctx)

    def iterate_gmres(self, K, k):
        check(self.lib.biot_iterate_gmres(self.ctx, K, k), self.ctx)

    def iterate_cheb(self, K, m, alpha=30.0):
        check(self.lib.biot_iterate_cheb(self.ctx, int(K), int(m), float(alpha)), self.ctx)

    def iterate_gs_gmres(self, K, k):
        check(self.lib.biot_iterate_gs_gmres(self.ctx, K, k), self.ctx)

    def gs_begin(self, K, gmres_k=0):
        check(self.lib.biot_gs_begin_gmres(self.ctx, K, gmres_k), self.ctx)
        n = ctypes.c_int32()
        check(self.lib.biot_gs_waves(self.ctx, ctypes.byref(n)), self.ctx)
        return n.value

    def gs_wave(self):
        check(self.lib.biot_gs_wave(self.ctx), self.ctx)

    def gs_end(self):
        check(self.lib.biot_gs_end(self.ctx), self.ctx)

    def iterate(self, K):
        check(self.lib.biot_iterate(self.ctx, int(K)), self.ctx)

    def residual_norms(self):
        out = np.empty((self.n_tl, 2))
        check(self.lib.biot_residual_norms(self.ctx, ptr(out)), self.ctx)
        return out

    def residual_history(self, k):
        out = np.empty((self.n_tl, 2))
        check(self.lib.biot_residual_history(self.ctx, int(k), ptr(out)), self.ctx)
        return out

    def solution(self, n=None, count=None):
        n = self.first_step if n is None else n
        count = (self.first_step + self.n_tl - n) if count is None else count
        out = np.empty((count, self.ndof))
        check(self.lib.biot_solution(self.ctx, n, count, ptr(out)), self.ctx)
        return out

    def last_slice(self):
        out = np.empty(self.ndof)
        check(self.lib.biot_last_slice(self.ctx, ptr(out)), self.ctx)
        return out

    def set_ghost(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        check(self.lib.biot_set_ghost(self.ctx, ptr(x)), self.ctx)

    def last_timing(self):
        out = np.zeros(2)
        check(self.lib.biot_last_timing(self.ctx, ptr(out)), self.ctx)
        return out

    def close(self):
        if self.ctx:
            self.lib.biot_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(_lib.load().biot_nccl_unique_id(buf))
    return buf.raw
