"""B200-native PCGM hot path for LQ optimal control of K x N grids (arXiv 2304.04980).

Drop-in for the reference package ``gridlq``'s solver path: the problem data model
(``GridLQProblem``...), ``pcg_solve`` / ``cg_solve`` / ``SolveReport`` and the operator /
preconditioner duck types, executed by hand-written sm_100a CUDA in libgridlq_b200.so.
"""

from .errors import (BreakdownError, DimensionGuardError, DimensionMismatchError, GridLQError,
                     MaxIterationsExceeded, NotPositiveDefiniteError)
from .problem import (BoundaryData, ConstSeq, GridArrays, GridLayout, GridLQProblem,
                      SubsystemData, arrays_from_problem, arrays_to_problem, boundary_arrays,
                      load_problem, problem_from_dict, problem_to_dict, rhs_offset_device,
                      save_problem, validate_arrays)
from .recovery import TrajectorySolution, kkt_residual, recover_solution
from .slab import SlabComm, SlabPcg, pcg_solve_slabs
from .solver import (COUNT_KEYS, GpuNestedJacobiPreconditioner, GpuSchurOperator, SolveReport,
                     apply_delta, build_schur, cg_solve, nbjm_solve, pcg_solve)

NestedJacobiPreconditioner = GpuNestedJacobiPreconditioner
SchurOperator = GpuSchurOperator

__all__ = [
    "BoundaryData", "BreakdownError", "COUNT_KEYS", "ConstSeq", "DimensionGuardError",
    "DimensionMismatchError", "GpuNestedJacobiPreconditioner", "GpuSchurOperator",
    "GridArrays", "GridLQError", "GridLQProblem", "GridLayout", "MaxIterationsExceeded",
    "NestedJacobiPreconditioner", "NotPositiveDefiniteError", "SchurOperator", "SolveReport",
    "SubsystemData", "apply_delta", "arrays_from_problem", "arrays_to_problem", "build_schur",
    "cg_solve", "nbjm_solve", "pcg_solve", "validate_arrays", "TrajectorySolution", "recover_solution",
    "kkt_residual", "load_problem", "save_problem", "problem_from_dict", "problem_to_dict",
    "SlabComm", "SlabPcg", "pcg_solve_slabs",
]

__version__ = "0.1.0"
