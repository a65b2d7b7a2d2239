"""B200-native hot path of arXiv 2310.10430 (parallel-in-time preconditioned Biot solver).

The product is libbiot_pit.so (include/biot_pit.h): host assembly + sm_100a fp64
kernels + NCCL time-slab halo.  This package is its thin Python binding.
"""
from .solver import BiotSolver, assemble_host, nccl_unique_id
from ._lib import BiotError, EXPORTS, LIB_PATH, FLAG_MANUAL_HALO, FLAG_NO_GRAPH, FLAG_DEFER_STEP0, FLAG_SWEEP_SLABS

__all__ = ["BiotSolver", "assemble_host", "nccl_unique_id", "BiotError", "EXPORTS", "LIB_PATH",
           "FLAG_MANUAL_HALO", "FLAG_NO_GRAPH", "FLAG_DEFER_STEP0", "FLAG_SWEEP_SLABS"]
