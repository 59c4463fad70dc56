"""B200-native drop-in for the hot path of the reference qDSE solver (dsegap,
arXiv 2012.03667): the successive-approximation self-energy sweep.

Public names mirror /root/reference/pkg/src/dsegap/__init__.py:9-51 for the
hot path (solve, iterate_once, interp_*, build_grid, ModelParams, VARIANTS,
the error classes).  Numerics run in libdse_b200.so (hand-written sm_100a
CUDA, fp64) through the C ABI in include/dse_b200.h; there is no CPU fallback.
"""
from .errors import (ConsistencyError, DegenerateMomentumError, ExecutionEnvironmentError,
                     GridConstructionError, KinematicSingularityError, NumericalFailureError,
                     ParameterError)
from .grid import MomentumGrid, build_grid, merge_bracket_indices
from .harness import BenchReport, BenchRow, format_table, run_bench
from .interpolation import (ComparisonCounter, InterpStrategy, interp_indexed, interp_indexed_many,
                            interp_linear_batch, interp_search, interp_search_many)
from .iteration import successive_approximation
from .kernels import ModelParams, row_rhs
from .quadrature import QuadratureRule, gauss_chebyshev2, gauss_legendre
from .solver import (DEFAULT_PROBES_LOG10P, VARIANTS, AlgorithmVariant, Arithmetic, ExecutionMode,
                     GpuSweeper, IterationRecord, PropagatorSolution, iterate_once, resolve_gpus, resolve_threads,
                     solve, solve_batch)

__version__ = "0.1.0"

__all__ = [
    "ConsistencyError", "DegenerateMomentumError", "ExecutionEnvironmentError", "GridConstructionError",
    "KinematicSingularityError", "NumericalFailureError", "ParameterError",
    "MomentumGrid", "build_grid", "merge_bracket_indices",
    "BenchReport", "BenchRow", "format_table", "run_bench",
    "ComparisonCounter", "InterpStrategy", "interp_indexed", "interp_indexed_many", "interp_linear_batch",
    "interp_search", "interp_search_many",
    "successive_approximation", "ModelParams", "row_rhs",
    "QuadratureRule", "gauss_chebyshev2", "gauss_legendre",
    "DEFAULT_PROBES_LOG10P", "VARIANTS", "AlgorithmVariant", "Arithmetic", "ExecutionMode", "GpuSweeper",
    "IterationRecord", "PropagatorSolution", "iterate_once", "resolve_gpus", "resolve_threads", "solve", "solve_batch",
]
