"""Tolerance families (mirrors matexpo/tolerances.py:11-36) plus the
relative-Frobenius tolerance that scales with log2 k."""

from __future__ import annotations

import math

from .dtypes import DType

VECTORIZED_SAFETY = 8
ASSOCIATIVITY_SAFETY = 8
ORACLE_SAFETY = 64
DEVICE_SAFETY = 64
FRO_SAFETY = 16


def _u(dtype) -> float:
    if isinstance(dtype, DType):
        return dtype.roundoff
    return 2.0 ** -24 if str(dtype) in ("float32", "f32") else 2.0 ** -53


def vectorized_tol(n: int, dtype) -> float:
    return n * _u(dtype) * VECTORIZED_SAFETY


def associativity_tol(n: int, dtype) -> float:
    return n * n * _u(dtype) * ASSOCIATIVITY_SAFETY


def oracle_tol(power: int, n: int, dtype) -> float:
    """max_rel bound, square-and-multiply vs repeated multiply (tolerances.py:311-313)."""
    return power * n * _u(dtype) * ORACLE_SAFETY


def device_tol(n: int, dtype) -> float:
    """Per-multiply max_rel bound for device backends (tolerances.py:316-319)."""
    return n * _u(dtype) * DEVICE_SAFETY


def multiply_count(power: int) -> int:
    return power.bit_length() - 1 + bin(power).count("1") - 1 if power >= 1 else 0


def fro_tol(n: int, power: int, dtype) -> float:
    """Relative-Frobenius bound for A^power vs the CPU oracle:
    16 * m(k) * sqrt(n) * u, m(k) = floor(log2 k) + popcount(k) - 1 (~ log2 k).
    Calibrated in SURVEY §8(d) (worst observed ratio 6.24 for the reference
    fp32 chain against its fp64 chain)."""
    return FRO_SAFETY * max(multiply_count(power), 1) * math.sqrt(n) * _u(dtype)


def fro_tol_conditioned(n: int, power: int, dtype) -> float:
    """The stated fallback 16 * (m(k) * sqrt(n) + k) * u for inputs whose
    ~k*u conditioning of A -> A^k exceeds the log2 k form."""
    return FRO_SAFETY * (max(multiply_count(power), 1) * math.sqrt(n) + power) * _u(dtype)
