"""B200-native iteration engine for the UV-decomposition ADMM conic solver.

Drop-in for the reference package ``conefree`` (arXiv 2203.05027): the same
``solve(p, cfg=None, init=None) -> SolveResult`` API and problem types, with
the iteration loop (solver.py:312-327) running as hand-written sm_100a fp64
kernels in ``libcfb200.so``. Importing the package needs no
GPU; creating a plan (``solve``) does, and fails loudly without one.
"""

from .api import (
    IterationReport,
    SolveResult,
    SolverConfig,
    SolverState,
    check_termination,
    solve,
    solve_batch,
)
from .binio import (
    TRACE_COLUMNS,
    ParseError,
    parse_problem,
    read_problem,
    read_problem_binary,
    write_problem,
    write_problem_binary,
    write_problem_file,
    write_solution,
    write_solution_file,
    trace_csv,
)
from .engine import DevicePlan
from .instances import GeneratedInstance, GenSpec, generate, generate_witnessed, shape_for_nnz
from .problem import ConeSpec, ProblemInstance, TripletMatrix, ValidationReport, validate

__version__ = "0.1.0"

__all__ = [
    "ConeSpec",
    "DevicePlan",
    "GenSpec",
    "GeneratedInstance",
    "IterationReport",
    "ParseError",
    "ProblemInstance",
    "SolveResult",
    "SolverConfig",
    "SolverState",
    "TripletMatrix",
    "ValidationReport",
    "check_termination",
    "parse_problem",
    "read_problem",
    "read_problem_binary",
    "write_problem",
    "write_problem_binary",
    "write_problem_file",
    "write_solution",
    "write_solution_file",
    "trace_csv",
    "TRACE_COLUMNS",
    "generate",
    "generate_witnessed",
    "shape_for_nnz",
    "solve",
    "solve_batch",
    "validate",
]
