"""Dense square matrices and error metrics (mirrors matexpo/linalg.py).

`Matrix` keeps the reference's contract (linalg.py:27-74): immutable,
square, row-major (element (i, j) at flat index i*n + j), float32 or
float64, C-contiguous, backing array frozen.  `compare` restates the
reference metrics (linalg.py:209-232).  There is deliberately no host
multiply here: every product goes through the sm_100a engine.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Iterable, Sequence, TextIO, Union

import numpy as np

from .dtypes import DType
from .errors import InvalidDimensionError, ShapeError


class Matrix:
    """Immutable dense square matrix with row-major storage."""

    __slots__ = ("array",)

    def __init__(self, array, copy: bool = True):
        arr = np.array(array, order="C", copy=True) if copy else np.asarray(array)
        if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
            raise ShapeError(f"expected a square 2-D array, got shape {arr.shape}")
        if arr.shape[0] < 1:
            raise InvalidDimensionError("matrix order must be >= 1")
        try:
            DType.of(arr)
        except ValueError as exc:
            raise ShapeError(str(exc)) from None
        if not arr.flags.c_contiguous:
            arr = np.ascontiguousarray(arr)
        arr.setflags(write=False)
        object.__setattr__(self, "array", arr)

    def __setattr__(self, name, value):
        raise AttributeError("Matrix is immutable")

    @property
    def n(self) -> int:
        return self.array.shape[0]

    @property
    def dtype(self) -> DType:
        return DType.of(self.array)

    @property
    def data(self) -> np.ndarray:
        return self.array.reshape(-1)

    @classmethod
    def from_rows(cls, rows: Sequence[Iterable[float]], dtype: DType = DType.F64) -> "Matrix":
        return cls(np.array([list(r) for r in rows], dtype=dtype.np))

    def astype(self, dtype: DType) -> "Matrix":
        if dtype is self.dtype:
            return self
        return Matrix(self.array.astype(dtype.np))

    def __repr__(self) -> str:
        return f"Matrix(n={self.n}, dtype={self.dtype.value})"


@dataclass(frozen=True)
class ErrorMetrics:
    """Elementwise and Frobenius error of a result against a reference."""

    max_abs: float
    max_rel: float
    frobenius_rel: float

    def __iter__(self):
        return iter((self.max_abs, self.max_rel, self.frobenius_rel))


def as_array(m) -> np.ndarray:
    """The row-major ndarray behind a Matrix (ours or the reference's) or an array."""
    arr = getattr(m, "array", m)
    return np.asarray(arr)


def wrap_like(template, arr: np.ndarray):
    """Wrap a result in the caller's matrix type (reference Matrix interop)."""
    cls = type(template)
    if cls is np.ndarray:
        return arr
    try:
        return cls(arr, copy=False)
    except TypeError:
        return Matrix(arr, copy=False)


def check_pair(a, b) -> None:
    aa, bb = as_array(a), as_array(b)
    if aa.shape != bb.shape:
        raise ShapeError(f"matrix orders differ: {aa.shape[0]} vs {bb.shape[0]}")
    if aa.dtype != bb.dtype:
        raise ShapeError(f"matrix dtypes differ: {aa.dtype} vs {bb.dtype}")


def identity(n: int, dtype: DType = DType.F64) -> Matrix:
    """The n-by-n multiplicative unit (A^0, expo.py:128-129)."""
    if n < 1:
        raise InvalidDimensionError(f"matrix order must be >= 1, got {n}")
    return Matrix(np.eye(n, dtype=dtype.np), copy=False)


def zeros(n: int, dtype: DType = DType.F64) -> Matrix:
    if n < 1:
        raise InvalidDimensionError(f"matrix order must be >= 1, got {n}")
    return Matrix(np.zeros((n, n), dtype=dtype.np), copy=False)


def compare(result, reference) -> ErrorMetrics:
    """max_abs, max_rel (= max_abs / max|ref|) and relative Frobenius error, in f64."""
    check_pair(result, reference)
    res = as_array(result).astype(np.float64)
    ref = as_array(reference).astype(np.float64)
    diff = np.abs(res - ref)
    max_abs = float(diff.max())
    denom = float(np.abs(ref).max())
    max_rel = (0.0 if max_abs == 0.0 else math.inf) if denom == 0.0 else max_abs / denom
    fro_ref = float(np.sqrt(np.sum(ref * ref)))
    fro_diff = float(np.sqrt(np.sum(diff * diff)))
    fro = (0.0 if fro_diff == 0.0 else math.inf) if fro_ref == 0.0 else fro_diff / fro_ref
    return ErrorMetrics(max_abs, max_rel, fro)


# --- text file format (linalg.py:235-276) -------------------------------------
# Line 1: "<n> <dtype>" with dtype in {f32, f64}; then n lines of n decimal
# values, row-major, shortest round-trip repr; reading back is bitwise exact.

def write_matrix(m, dest: Union[str, os.PathLike, TextIO]) -> None:
    arr = as_array(m)
    if hasattr(dest, "write"):
        _write_stream(arr, dest)
    else:
        with open(dest, "w", encoding="utf-8") as fh:
            _write_stream(arr, fh)


def _write_stream(arr: np.ndarray, fh: TextIO) -> None:
    fh.write(f"{arr.shape[0]} {DType.of(arr).value}\n")
    for row in arr:
        fh.write(" ".join(str(v) for v in row))
        fh.write("\n")


def read_matrix(src: Union[str, os.PathLike, TextIO]) -> Matrix:
    if hasattr(src, "read"):
        return _read_stream(src)
    with open(src, "r", encoding="utf-8") as fh:
        return _read_stream(fh)


def _read_stream(fh: TextIO) -> Matrix:
    header = fh.readline().split()
    if len(header) != 2:
        raise ShapeError("matrix file header must be '<n> <dtype>'")
    n = int(header[0])
    dtype = DType.parse(header[1])
    if n < 1:
        raise InvalidDimensionError(f"matrix order must be >= 1, got {n}")
    out = np.empty((n, n), dtype=dtype.np)
    for i in range(n):
        parts = fh.readline().split()
        if len(parts) != n:
            raise ShapeError(f"row {i} has {len(parts)} values, expected {n}")
        out[i] = [dtype.np(float(tok)) for tok in parts]
    return Matrix(out, copy=False)
