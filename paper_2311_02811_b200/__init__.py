"""B200-native (sm_100a) Contour connected components -- the hot path of
arXiv 2311.02811's reference package ``minmapcc`` rebuilt as hand-written
CUDA behind a C-ABI (include/contour.h), with the reference's Python entry
points (engine.py) mirrored here as a drop-in."""

from .engine import (
    VARIANTS,
    ForestDiagnostics,
    IterationStats,
    LabelArray,
    Schedule,
    canonical_variant,
    conditional_min_assign,
    early_convergence_check,
    forest_diagnostics,
    make_schedule,
    mm_order,
    run_contour,
)
from .errors import IterationCapExceeded

__version__ = "0.1.0"

__all__ = [
    "VARIANTS", "ForestDiagnostics", "IterationStats", "LabelArray", "Schedule",
    "canonical_variant", "conditional_min_assign", "early_convergence_check",
    "forest_diagnostics", "make_schedule", "mm_order", "run_contour", "IterationCapExceeded",
    "__version__",
]
