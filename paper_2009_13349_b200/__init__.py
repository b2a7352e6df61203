"""tccd: B200-native batched Tight-Inclusion CCD (arXiv 2009.13349).

The hot path of the reference package ccdkit -- the inclusion-based
conservative root finder (pkg/src/ccdkit/_kernel.py:136 solve_kernel, called
through solver.solve, pkg/src/ccdkit/solver.py:50) -- rebuilt as sm_100a
FP64 CUDA kernels behind a C-ABI (include/tccd.h, csrc/), with the
reference's solve-side Python surface on top.
"""

from .core import CCDResult, DomainBox, Query, QueryKind, SolverConfig
from .inclusion import FilterEps, compute_filters, compute_gamma
from .solver import OUTPUT_FIELDS, shard_bounds, solve, solve_batch, solve_kernel, warm_up
from .baselines import irf_batch, irf_solve

__all__ = [
    "CCDResult", "DomainBox", "FilterEps", "OUTPUT_FIELDS", "Query", "QueryKind",
    "SolverConfig", "compute_filters", "compute_gamma", "shard_bounds", "solve",
    "solve_batch", "solve_kernel", "warm_up", "irf_batch", "irf_solve",
]
