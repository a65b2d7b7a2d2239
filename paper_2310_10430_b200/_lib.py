"""ctypes binding of include/biot_pit.h (argument marshalling only).

Every computation happens inside libbiot_pit.so (host assembly + sm_100a
kernels).  There is no Python or CPU fallback: if the library is missing this
module raises, and on a machine without a B200 biot_setup fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# BIOT_LIB_OVERRIDE: load another build of the library (kernel-variant experiments only)
LIB_PATH = os.environ.get("BIOT_LIB_OVERRIDE") or os.path.join(HERE, "libbiot_pit.so")

_d = ctypes.POINTER(ctypes.c_double)
_i32 = ctypes.POINTER(ctypes.c_int32)
_i64 = ctypes.POINTER(ctypes.c_int64)
_u8 = ctypes.POINTER(ctypes.c_uint8)

BIOT_OK = 0
STATUS = {0: "BIOT_OK", 1: "BIOT_E_INVALID", 2: "BIOT_E_NOMEM", 3: "BIOT_E_CUDA",
          4: "BIOT_E_NCCL", 5: "BIOT_E_STATE", 6: "BIOT_E_NONFINITE"}
FLAG_MANUAL_HALO = 1
FLAG_NO_GRAPH = 2
FLAG_DEFER_STEP0 = 4
FLAG_SWEEP_SLABS = 8


class BiotMesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n_nodes", ctypes.c_int64), ("coords", _d),
                ("n_cells", ctypes.c_int64), ("cells", _i32)]


class BiotMaterial(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("mu", ctypes.c_double), ("alpha", ctypes.c_double),
                ("storage", ctypes.c_double), ("kappa", _d), ("kappa_uniform", ctypes.c_double),
                ("beta", ctypes.c_double), ("h", ctypes.c_double)]


# void (*source_eval)(int32_t q, int64_t npts, const double *xyz, double *vals, void *user)
SOURCE_EVAL = ctypes.CFUNCTYPE(None, ctypes.c_int32, ctypes.c_int64, _d, _d, ctypes.c_void_p)


class BiotBC(ctypes.Structure):
    _fields_ = [("dirichlet", _u8), ("n_traction_facets", ctypes.c_int64),
                ("traction_facets", _i32), ("traction", ctypes.c_double * 3),
                ("load_scale", _d), ("x_initial", _d), ("n_sources", ctypes.c_int32),
                ("source_eval", SOURCE_EVAL), ("source_user", ctypes.c_void_p), ("source_coef", _d),
                ("dirichlet_values", _d), ("dirichlet_coef", _d)]


class BiotOpts(ctypes.Structure):
    _fields_ = [("precond", ctypes.c_int32), ("omega", ctypes.c_double), ("device", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("stream", ctypes.c_void_p), ("flags", ctypes.c_uint32), ("history", ctypes.c_int32)]


class BiotInfo(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n_comp", ctypes.c_int32), ("n_nodes", ctypes.c_int64),
                ("n_dof", ctypes.c_int64), ("n_t", ctypes.c_int32), ("n_t_local", ctypes.c_int32),
                ("first_step", ctypes.c_int32), ("iterations", ctypes.c_int64),
                ("kernel_path", ctypes.c_int32), ("n_slots", ctypes.c_int32), ("beta", ctypes.c_double),
                ("bytes_per_iter", ctypes.c_double), ("flops_per_iter", ctypes.c_double),
                ("device_bytes", ctypes.c_double), ("launches_per_iter", ctypes.c_int32),
                ("interior_nodes", ctypes.c_int32), ("comm_nranks", ctypes.c_int32), ("graph", ctypes.c_int32)]


# every symbol include/biot_pit.h declares (checked by tests/test_abi.py)
EXPORTS = ["biot_setup", "biot_set_iterate", "biot_set_load_scale", "biot_iterate", "biot_iterate_gs", "biot_iterate_gmres", "biot_iterate_cheb",
           "biot_iterate_gs_gmres", "biot_gs_begin_gmres",
           "biot_gs_begin", "biot_gs_waves", "biot_gs_wave", "biot_gs_end",
           "biot_residual_norms", "biot_residual_history", "biot_solution", "biot_last_slice",
           "biot_set_ghost", "biot_assemble_host", "biot_assemble_loads_host", "biot_get_info", "biot_last_timing",
           "biot_nccl_unique_id", "biot_destroy", "biot_last_error", "biot_status_string",
           "biot_abi_version", "biot_mesh_structured", "biot_bc_column", "biot_free"]

_lib = None


def load():
    """Load (building first if stale) libbiot_pit.so and declare signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _b
        _b.build()
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    ctx_p = ctypes.c_void_p
    S = ctypes.c_int
    L.biot_setup.argtypes = [P(BiotMesh), P(BiotMaterial), P(BiotBC), ctypes.c_double, ctypes.c_int32,
                             P(BiotOpts), P(ctx_p)]
    L.biot_set_iterate.argtypes = [ctx_p, ctypes.c_int32, ctypes.c_int32, _d]
    L.biot_set_load_scale.argtypes = [ctx_p, _d]
    L.biot_iterate.argtypes = [ctx_p, ctypes.c_int32]
    L.biot_iterate_gs.argtypes = [ctx_p, ctypes.c_int32]
    L.biot_iterate_gmres.argtypes = [ctx_p, ctypes.c_int32, ctypes.c_int32]
    L.biot_iterate_gs_gmres.argtypes = [ctx_p, ctypes.c_int32, ctypes.c_int32]
    L.biot_iterate_cheb.argtypes = [ctx_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_double]
    L.biot_gs_begin_gmres.argtypes = [ctx_p, ctypes.c_int32, ctypes.c_int32]
    L.biot_gs_begin.argtypes = [ctx_p, ctypes.c_int32]
    L.biot_gs_waves.argtypes = [ctx_p, ctypes.POINTER(ctypes.c_int32)]
    L.biot_gs_wave.argtypes = [ctx_p]
    L.biot_gs_end.argtypes = [ctx_p]
    L.biot_residual_norms.argtypes = [ctx_p, _d]
    L.biot_residual_history.argtypes = [ctx_p, ctypes.c_int64, _d]
    L.biot_solution.argtypes = [ctx_p, ctypes.c_int32, ctypes.c_int32, _d]
    L.biot_last_slice.argtypes = [ctx_p, _d]
    L.biot_set_ghost.argtypes = [ctx_p, _d]
    L.biot_assemble_host.argtypes = [P(BiotMesh), P(BiotMaterial), P(BiotBC), ctypes.c_double,
                                     _i64, _i64, _i64, _d, _i64, _i64, _i64, _d, _d, _d]
    L.biot_assemble_loads_host.argtypes = [P(BiotMesh), P(BiotMaterial), P(BiotBC), ctypes.c_double,
                                           P(ctypes.c_int32), _d, P(ctypes.c_int32), P(ctypes.c_int32)]
    L.biot_mesh_structured.argtypes = [ctypes.c_int32, ctypes.c_int32, P(_d), P(_i32), _i64, _i64]
    L.biot_bc_column.argtypes = [P(BiotMesh), ctypes.c_double, _u8, _d, _i64, _i32]
    L.biot_free.argtypes = [ctypes.c_void_p]
    L.biot_free.restype = None
    L.biot_get_info.argtypes = [ctx_p, P(BiotInfo)]
    L.biot_last_timing.argtypes = [ctx_p, _d]
    L.biot_nccl_unique_id.argtypes = [ctypes.c_void_p]
    L.biot_destroy.argtypes = [ctx_p]
    L.biot_destroy.restype = None
    L.biot_last_error.argtypes = [ctx_p]
    L.biot_last_error.restype = ctypes.c_char_p
    L.biot_status_string.argtypes = [ctypes.c_int]
    L.biot_status_string.restype = ctypes.c_char_p
    L.biot_abi_version.restype = ctypes.c_int32
    for name in EXPORTS:
        f = getattr(L, name)
        if f.restype is ctypes.c_int and name not in ("biot_abi_version",):
            f.restype = S
    _lib = L
    return L


class BiotError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def check(status, ctx=None):
    if status != BIOT_OK:
        msg = load().biot_last_error(ctx)
        raise BiotError(status, msg.decode() if msg else "")


def ptr(a, t=_d):
    return None if a is None else a.ctypes.data_as(t)


class Inputs:
    """Owns the contiguous numpy arrays behind the ABI structs of one problem."""

    def __init__(self, prob, load_scale=None, x_initial=None, beta=None):
        self.coords = np.ascontiguousarray(prob.coords, dtype=np.float64)
        self.cells = np.ascontiguousarray(prob.cells, dtype=np.int32)
        self.kappa = np.ascontiguousarray(np.broadcast_to(prob.kappa, (self.cells.shape[0],)),
                                          dtype=np.float64)
        self.dirichlet = np.ascontiguousarray(prob.dirichlet, dtype=np.uint8)
        self.facets = np.ascontiguousarray(prob.facets, dtype=np.int32)
        self.load_scale = None if load_scale is None else np.ascontiguousarray(load_scale, dtype=np.float64)
        if x_initial is None:
            x_initial = getattr(prob, "x_initial", None)
        self.x_initial = None if x_initial is None else np.ascontiguousarray(x_initial, dtype=np.float64)
        d = prob.dim
        self.mesh = BiotMesh(d, self.coords.shape[0], ptr(self.coords), self.cells.shape[0],
                             ptr(self.cells, _i32))
        self.mat = BiotMaterial(prob.lam, prob.mu, prob.alpha, prob.storage, ptr(self.kappa), 0.0,
                                -1.0 if beta is None else beta, prob.h)
        tr = (ctypes.c_double * 3)(*([float(v) for v in prob.traction] + [0.0] * (3 - d)))
        # time-dependent sources and Dirichlet data (§4.1; optional Problem fields):
        # prob.source_fn(q, xyz [npts, d]) -> [npts, d+1] is evaluated by the library at its
        # quadrature points through the source_eval callback
        fn = getattr(prob, "source_fn", None)
        n_src = 0 if fn is None else int(prob.n_sources)
        self.source_coef = None if fn is None else np.ascontiguousarray(prob.source_coef, dtype=np.float64)
        self.cb_error = None

        def _eval(q, npts, xyz, vals, user):
            try:
                X = np.ctypeslib.as_array(xyz, shape=(npts, d))
                V = np.ctypeslib.as_array(vals, shape=(npts, d + 1))
                V[:] = fn(q, X)
            except Exception as e:      # leave NaNs: the library rejects them
                self.cb_error = e

        self.source_eval = SOURCE_EVAL(_eval) if fn is not None else SOURCE_EVAL()
        dv = getattr(prob, "dirichlet_values", None)
        self.dirichlet_values = None if dv is None else np.ascontiguousarray(dv, dtype=np.float64)
        dc = getattr(prob, "dirichlet_coef", None)
        self.dirichlet_coef = None if dc is None else np.ascontiguousarray(dc, dtype=np.float64)
        self.bc = BiotBC(ptr(self.dirichlet, _u8), self.facets.shape[0], ptr(self.facets, _i32), tr,
                         ptr(self.load_scale), ptr(self.x_initial), n_src, self.source_eval, None,
                         ptr(self.source_coef), ptr(self.dirichlet_values), ptr(self.dirichlet_coef))
