"""Seeded synthetic workloads (inputs only; no arithmetic of the method)."""
from .generators import (Problem, make_problem, mesh, mesh_square, mesh_cube, column_dirichlet,
                         top_facets, kappa_cells, initial_iterate, load_scales, std_normal,
                         uniform01, sm64, trig_problem, linear_patch_problem, trig_source, trig_exact,
                         patch_exact,
                         all_boundary_dirichlet, lame_from_young)
from .configs import CONFIGS, DESCRIPTIONS, config_problem

__all__ = ["Problem", "make_problem", "mesh", "mesh_square", "mesh_cube", "column_dirichlet",
           "top_facets", "kappa_cells", "initial_iterate", "load_scales", "std_normal",
           "uniform01", "sm64", "CONFIGS", "DESCRIPTIONS", "config_problem", "trig_problem",
           "linear_patch_problem", "trig_source", "trig_exact", "patch_exact", "all_boundary_dirichlet", "lame_from_young"]
