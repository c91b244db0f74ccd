"""Deterministic inputs generated on the device (next-row f3 of SURVEY §8(f)).

``random_matrix`` is bit-identical to the reference's SplitMix64
``random_matrix`` (linalg.py:109-148); ``scaled_batch`` is the configs'
spectrally normalised recipe fl(random_matrix(n, F64, seed0 + i) * sqrt(12/n))
(SURVEY §8(d)).  Both run as one sm_100a kernel and only the result crosses
PCIe.
"""

from __future__ import annotations

import math

import numpy as np

from .dtypes import DType
from .errors import InvalidDimensionError, InvalidRangeError
from .linalg import Matrix


def _gen(n: int, batch: int, dtype: DType, seed0: int, lo: float, hi: float, scale: float,
         device: int) -> np.ndarray:
    if n < 1:
        raise InvalidDimensionError(f"matrix order must be >= 1, got {n}")
    if not lo < hi:
        raise InvalidRangeError(f"need lo < hi, got [{lo}, {hi})")
    from .engine import default_engine

    eng = default_engine(device)
    out = np.empty((batch, n, n), dtype=dtype.np)
    d = eng.alloc(out.nbytes)
    try:
        eng.random_device(d, n, batch, seed0, lo, hi, scale, dtype.mode)
        eng.download(out, d)
    finally:
        eng.free(d)
    return out


def splitmix64(seed: int, count: int, device: int = 0) -> np.ndarray:
    """First ``count`` outputs of SplitMix64 seeded with ``seed`` (linalg.py:117-124),
    as uint64, generated on the device; bit-identical to the reference."""
    if count < 0:
        raise InvalidDimensionError(f"count must be >= 0, got {count}")
    from .engine import default_engine

    out = np.empty(count, dtype=np.uint64)
    if count == 0:
        return out
    eng = default_engine(device)
    d = eng.alloc(out.nbytes)
    try:
        eng.splitmix64_device(d, seed, count)
        eng.download(out, d)
    finally:
        eng.free(d)
    return out


def random_matrix(n: int, dtype: DType = DType.F64, seed: int = 0, lo: float = -0.5,
                  hi: float = 0.5, device: int = 0) -> Matrix:
    """Deterministic uniform matrix in [lo, hi) (linalg.py:127-148), bit-exact."""
    return Matrix(_gen(n, 1, dtype, seed, lo, hi, 0.0, device)[0], copy=False)


def scaled_batch(n: int, batch: int, dtype: DType = DType.F32, seed0: int = 42,
                 device: int = 0) -> np.ndarray:
    """(batch, n, n) stack, element i = fl(random_matrix(n, F64, seed0+i) * sqrt(12/n))."""
    return _gen(n, batch, dtype, seed0, -0.5, 0.5, math.sqrt(12.0 / n), device)


def scaled_input(n: int, dtype: DType = DType.F32, seed: int = 42, device: int = 0) -> Matrix:
    return Matrix(scaled_batch(n, 1, dtype, seed, device)[0], copy=False)
