"""Exception types, mirroring matexpo/errors.py (names, bases, attributes) and
the device errors of gpu-backend/src/errors.ts, mapped from the C-ABI status
codes of include/matexpo_b200.h.
"""


class MatexpoError(Exception):
    """Base class for all errors raised by this package."""


class InvalidDimensionError(MatexpoError, ValueError):
    """Matrix order is not a positive integer."""


class InvalidRangeError(MatexpoError, ValueError):
    """Element range [lo, hi) is empty or inverted."""


class ShapeError(MatexpoError, ValueError):
    """Operands disagree in order or element dtype."""


class UnsupportedPowerError(MatexpoError, ValueError):
    """The repeated-multiply baseline has no notion of this power."""


class ValidationError(MatexpoError, ValueError):
    """Rejected by the C-ABI before any device work (errors.ts ValidationError)."""


class UnsupportedError(MatexpoError, ValueError):
    """Mode or size outside what the sm_100a kernels support."""


class BackendStepError(MatexpoError, RuntimeError):
    """A backend multiply failed; carries the plan step index (errors.py:43-49)."""

    def __init__(self, step_index: int, step_name: str, cause: Exception):
        self.step_index = step_index
        self.step_name = step_name
        super().__init__(f"backend multiply failed at step {step_index} ({step_name}): {cause}")


class DeviceUnavailableError(MatexpoError, RuntimeError):
    """No usable B200 (sm_100) device (errors.ts DeviceUnavailableError)."""


class DeviceError(MatexpoError, RuntimeError):
    """A CUDA (or NCCL) runtime failure inside the engine."""


class ExtensionNotBuiltError(MatexpoError, RuntimeError):
    """libmatexpo_b200.so is missing: there is no CPU fallback, build it."""


class ConfigError(MatexpoError, ValueError):
    """Benchmark configuration failed validation."""


class TableError(MatexpoError, ValueError):
    """The comparison table lacks a cell (errors.py:56 of the reference)."""
