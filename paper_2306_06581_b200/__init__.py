"""B200-native Spar-Sink hot path (arXiv 2306.06581).

The product is libspk_b200.so (CUDA kernels for sm_100a behind the C ABI in
include/spk.h) and libsparsink_b200.so (the C++ drop-in for the reference's
namespace sparsink entry points). This Python package is a thin ctypes
host mirror used by tests and bench.py; it has no CPU compute path.
"""
from .api import (  # noqa: F401
    ERRORS,
    Context,
    Coords,
    Dense,
    Result,
    Sketch,
    SolverConfig,
    SparSinkOptions,
    SparsinkError,
    default_context,
    sinkhorn_ot,
    sinkhorn_uot,
    spar_sink_ot,
    spar_sink_uot,
)

__all__ = [
    "ERRORS", "Context", "Coords", "Dense", "Result", "Sketch", "SolverConfig", "SparSinkOptions", "SparsinkError",
    "default_context", "sinkhorn_ot", "sinkhorn_uot", "spar_sink_ot", "spar_sink_uot",
]
