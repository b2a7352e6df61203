"""tccd: B200-native batched Tight-Inclusion CCD (arXiv 2009.13349).

The hot path of the reference package ccdkit -- the inclusion-based
conservative root finder (pkg/src/ccdkit/_kernel.py:136 solve_kernel, called
through solver.solve, pkg/src/ccdkit/solver.py:50) -- rebuilt as sm_100a
FP64 CUDA kernels behind a C-ABI (include/tccd.h, csrc/), with the
reference's solve-side Python surface on top.
"""

from .core import (CCDResult, DomainBox, Query, QueryKind, SolverConfig, Vec3, eval_F, eval_F_ee,
                   eval_F_vf)
from .inclusion import (BoxClass, FilterEps, InclusionBox, box_inclusion, box_inclusion_batch,
                        classify_box, compute_filters, compute_gamma, kappas, kappas_batch)
from .solver import (OUTPUT_FIELDS, queue_order, shard_bounds, solve, solve_batch, solve_kernel,
                     split, warm_up)
from .baselines import irf_batch, irf_solve
from .sharding import solve_devices, solve_sharded

__all__ = [
    "BoxClass", "CCDResult", "DomainBox", "FilterEps", "InclusionBox", "OUTPUT_FIELDS", "Query",
    "QueryKind", "SolverConfig", "Vec3", "box_inclusion", "box_inclusion_batch", "classify_box",
    "compute_filters", "compute_gamma", "eval_F", "eval_F_ee", "eval_F_vf", "kappas",
    "kappas_batch", "queue_order", "split", "shard_bounds", "solve",
    "solve_batch", "solve_kernel", "warm_up", "irf_batch", "irf_solve", "solve_devices",
    "solve_sharded",
]
