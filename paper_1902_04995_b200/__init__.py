"""B200-native batch 2D linear programming (Seidel / RGB, arXiv 1902.04995).

Drop-in for the reference's lp2d::solve_batch path; see DESIGN.md.
"""
from . import lp2d, reduction  # noqa: F401
from .lp2d import (  # noqa: F401
    Batch, BatchResult, BlockConfig, DeviceBatch, GenKind, PackedBatch, PackedResult,
    Permutation, Problem, SchedulerKind, Solution, Tolerance, derive_seed, gen, gen_mixed,
    identity_permutation, kernel_launches, lane_imbalance, replicate, shuffle, solve_batch, solve_device,
    PermSeed,
    solve_packed,
)
from .lp2d import ParseError, problem_from_text, to_text  # noqa: F401  (io.hpp)
from .reduction import (  # noqa: F401  (reduction.hpp, bench.hpp contention)
    ContentionRecord, ReduceStrategy, contention_bench, segmented_extremes,
)

__all__ = [n for n in dir() if not n.startswith("_")]
