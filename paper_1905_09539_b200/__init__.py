"""B200-native Schur-basis solve of the tsylv reference (arXiv 1905.09539).

The hot path (forward transforms, reduced quasi-triangular solve, back
transforms) runs in hand-written sm_100a kernels inside ``libtsylv_gpu.so``;
this package is the Python host mirror of the reference's API on top of it.
"""
from .api import (Arithmetic, GSylvProblem, LaplaceProblem, PhaseTimings, RandomStream,
                  SolveReport, SolverConfig, Strategy, dimension_error, factorization_error,
                  gpu_error, gsylv_merged, gsylv_recursive, laplace_merged, laplace_recursive,
                  make_problem, mode_multiply, oracle, qz, random_problem, residual, schur, screen_gsylv,
                  screen_laplace, singular_error, solve_gsylv, solve_gsylv_tri, solve_laplace,
                  solve_sylvester_tri)

__all__ = [
    "Arithmetic", "GSylvProblem", "LaplaceProblem", "PhaseTimings", "RandomStream", "SolveReport",
    "SolverConfig", "Strategy", "dimension_error", "factorization_error", "gpu_error",
    "gsylv_merged", "gsylv_recursive", "laplace_merged", "laplace_recursive", "make_problem",
    "mode_multiply", "oracle", "qz", "random_problem", "residual", "schur", "screen_gsylv", "screen_laplace",
    "singular_error", "solve_gsylv",
    "solve_gsylv_tri", "solve_laplace", "solve_sylvester_tri",
]
