"""B200-native POD-2G solve path (arXiv 2207.02543): batched fp64 PCG with the
POD two-grid preconditioner, hand-written sm_100a CUDA behind a C-ABI
(include/pod2g_b200.h).  See DESIGN.md."""
from . import _lib
from .solver import (BatchSolver, CsrMatrix, PodBasis, Pod2gPreconditioner, SolveReport,
                     analyze_pattern, pcg_solve, reduced_solve)

__all__ = ["BatchSolver", "CsrMatrix", "PodBasis", "Pod2gPreconditioner", "SolveReport",
           "analyze_pattern", "pcg_solve", "reduced_solve", "_lib"]
