"""Seeded synthetic workloads (inputs only; no arithmetic of the method)."""
from .generators import (Problem, make_problem, mesh, mesh_square, mesh_cube, column_dirichlet,
                         top_facets, kappa_cells, initial_iterate, load_scales, std_normal,
                         uniform01, sm64)
from .configs import CONFIGS, DESCRIPTIONS, config_problem

__all__ = ["Problem", "make_problem", "mesh", "mesh_square", "mesh_cube", "column_dirichlet",
           "top_facets", "kappa_cells", "initial_iterate", "load_scales", "std_normal",
           "uniform01", "sm64", "CONFIGS", "DESCRIPTIONS", "config_problem"]
