"""paper_1204_3052_b200 — a B200-native engine for integer matrix powers A^k.

Drop-in for the hot path of the reference `matexpo` package
(/root/reference/pkg/src/matexpo): the same public names for the plan,
the backend plugin and ``exponentiate``, backed by hand-written sm_100a
kernels (tcgen05 3xTF32, DMMA FP64) behind the C ABI in
include/matexpo_b200.h.  See DESIGN.md.
"""

from .dtypes import DType
from .errors import (
    BackendStepError,
    ConfigError,
    DeviceError,
    DeviceUnavailableError,
    ExtensionNotBuiltError,
    InvalidDimensionError,
    InvalidRangeError,
    MatexpoError,
    ShapeError,
    TableError,
    UnsupportedError,
    UnsupportedPowerError,
    ValidationError,
)
from .linalg import ErrorMetrics, Matrix, compare, identity, read_matrix, write_matrix, zeros
from .tolerances import (
    associativity_tol,
    device_tol,
    fro_tol,
    fro_tol_conditioned,
    multiply_count,
    oracle_tol,
    vectorized_tol,
)
from .expo import (
    B200Backend,
    Backend,
    CountingBackend,
    ExponentPlan,
    Step,
    Strategy,
    b200_backend,
    count_transfers,
    exponentiate,
    exponentiate_batched,
    exponentiate_multi,
    multiply_count_for,
    plan_exponentiation,
    repeated_exponentiate,
)
from .generate import random_matrix, scaled_batch, scaled_input, splitmix64

__version__ = "0.1.0"

__all__ = [
    "DType", "MatexpoError", "InvalidDimensionError", "InvalidRangeError", "ShapeError",
    "UnsupportedPowerError", "BackendStepError", "ConfigError", "ValidationError",
    "UnsupportedError", "TableError", "DeviceUnavailableError", "DeviceError", "ExtensionNotBuiltError",
    "Matrix", "ErrorMetrics", "identity", "zeros", "compare", "random_matrix", "read_matrix",
    "write_matrix", "splitmix64",
    "scaled_batch", "scaled_input", "vectorized_tol", "associativity_tol", "oracle_tol",
    "device_tol", "fro_tol", "fro_tol_conditioned", "multiply_count", "Step", "Strategy",
    "ExponentPlan", "plan_exponentiation", "Backend", "CountingBackend", "B200Backend",
    "b200_backend", "exponentiate", "exponentiate_batched", "exponentiate_multi",
    "repeated_exponentiate",
    "count_transfers", "multiply_count_for", "Engine", "__version__",
    # the reference's harness names (bench.py:40-98, :183-395), for the b200 backend
    "BenchConfig", "BenchmarkRecord", "make_backend", "run_benchmark", "emit_csv", "read_csv",
    "emit_table",
]

_HARNESS = ("BenchConfig", "BenchmarkRecord", "make_backend", "run_benchmark", "emit_csv",
            "read_csv", "emit_table")


def __getattr__(name):
    if name == "Engine":
        from .engine import Engine

        return Engine
    if name in _HARNESS:
        from . import harness

        return getattr(harness, name)
    if name in ("engine", "distributed", "build", "harness", "cli"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
