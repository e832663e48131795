"""B200-native GCG eigensolver hot path (drop-in for the reference `gcgeig` solver).

Public surface mirrors the reference (pkg/src/gcgeig/__init__.py):
``gcg_solve(a, b=None, config=None) -> SolverReport`` with ``SolverConfig``,
the B-orthogonalisation entry points and the MultiVec* ops — all executed by
hand-written sm_100a CUDA kernels in libgcgb200.so (C ABI: include/gcgb200.h).
"""

from .errors import (
    AllDependent,
    GcgError,
    InvalidMatrix,
    InvalidRange,
    InvalidShape,
    IoError,
    NoConvergence,
    ParseError,
    UnknownGenerator,
    Unsupported,
)
from .io import (
    RunRecord,
    generate_builtin,
    history_rows,
    read_matrix_market,
    write_history,
    write_matrix_market,
)
from .orth import OrthConfig, OrthOutcome, modified_block_orth, orth_against, recursive_orth_svd
from .solver import (
    IterationRecord,
    SolverConfig,
    SolverReport,
    gcg_solve,
    moving_memory_budget,
    select_shift,
)

__version__ = "0.1.0"

__all__ = [
    "gcg_solve",
    "SolverConfig",
    "SolverReport",
    "IterationRecord",
    "select_shift",
    "moving_memory_budget",
    "OrthConfig",
    "OrthOutcome",
    "recursive_orth_svd",
    "modified_block_orth",
    "orth_against",
    "GcgError",
    "InvalidMatrix",
    "InvalidShape",
    "InvalidRange",
    "NoConvergence",
    "AllDependent",
    "Unsupported",
    "ParseError",
    "UnknownGenerator",
    "IoError",
    "read_matrix_market",
    "write_matrix_market",
    "generate_builtin",
    "RunRecord",
    "write_history",
    "history_rows",
]
