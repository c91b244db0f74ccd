"""TEST INFRASTRUCTURE ONLY — CPU oracle for matrix exponentiation A^k.

A restatement of the reference `matexpo` hot path
(/root/reference/pkg/src/matexpo), used as the checker for the B200 engine:

* ``splitmix64`` / ``random_matrix``  — linalg.py:109-148
* ``matmul``  (== ``matmul_naive``)   — linalg.py:151-164 (ascending k, no FMA)
* ``plan``    (== ``plan_exponentiation``) — expo.py:60-75
* ``exponentiate``                    — expo.py:121-139
* ``compare``                         — linalg.py:209-232
* ``oracle_tol`` / ``device_tol``     — tolerances.py:18-36
* ``fro_tol`` — the relative-Frobenius tolerance of SURVEY.md §8(d)
* ``scaled_input`` — the spectrally normalised input recipe of SURVEY §8(d)

The arithmetic runs in oracle/matexpo_oracle.c (built by oracle/Makefile with
-ffp-contract=off); tests/test_oracle.py pins it bit-for-bit to the golden
vectors in tests/golden/, which tests/golden/make_golden.py produced by
importing the unmodified reference.  Parity status: PINNED.

Nothing in the product package imports this module.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Optional

import numpy as np

__all__ = [
    "lib",
    "splitmix64",
    "random_matrix",
    "scaled_input",
    "scaled_batch",
    "matmul",
    "matmul_rows",
    "plan",
    "multiply_count",
    "exponentiate",
    "exponentiate_batched",
    "matmul_mod",
    "exponentiate_mod",
    "compare",
    "oracle_tol",
    "device_tol",
    "fro_tol",
    "max_threads",
    "U32",
    "U64",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmatexpo_oracle.so")

U32 = 2.0 ** -24
U64 = 2.0 ** -53

_lib: Optional[ctypes.CDLL] = None


def _build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib() -> ctypes.CDLL:
    """Load (building if needed) the C oracle."""
    global _lib
    if _lib is not None:
        return _lib
    src = os.path.join(_HERE, "matexpo_oracle.c")
    if not os.path.exists(_SO) or (
        os.path.exists(src) and os.path.getmtime(src) > os.path.getmtime(_SO)
    ):
        _build()
    L = ctypes.CDLL(_SO)
    i64, u64, c_int, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
    L.mxo_splitmix64.argtypes = [u64, i64, vp]
    L.mxo_random_f64.argtypes = [i64, u64, ctypes.c_double, ctypes.c_double, vp]
    L.mxo_random_f32.argtypes = [i64, u64, ctypes.c_double, ctypes.c_double, vp]
    for name in ("mxo_matmul_f32", "mxo_matmul_f64"):
        getattr(L, name).argtypes = [i64, vp, vp, vp, c_int]
    for name in ("mxo_matmul_rows_f32", "mxo_matmul_rows_f64"):
        getattr(L, name).argtypes = [i64, i64, i64, vp, vp, vp, c_int]
    L.mxo_plan.argtypes = [i64, ctypes.c_char_p, i64]
    L.mxo_plan.restype = i64
    for name in ("mxo_exponentiate_f32", "mxo_exponentiate_f64"):
        getattr(L, name).argtypes = [i64, i64, vp, vp, c_int]
        getattr(L, name).restype = i64
    L.mxo_exponentiate_batched_f32.argtypes = [i64, i64, i64, vp, vp, c_int]
    L.mxo_exponentiate_batched_f32.restype = i64
    L.mxo_matmul_mod.argtypes = [i64, ctypes.c_uint32, vp, vp, vp, c_int]
    L.mxo_exponentiate_mod.argtypes = [i64, i64, ctypes.c_uint32, vp, vp, c_int]
    L.mxo_exponentiate_mod.restype = i64
    L.mxo_max_threads.restype = c_int
    _lib = L
    return L


def max_threads() -> int:
    return int(lib().mxo_max_threads())


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --- generation ------------------------------------------------------------

def splitmix64(seed: int, count: int) -> np.ndarray:
    """linalg.py:117-124."""
    out = np.empty(count, dtype=np.uint64)
    lib().mxo_splitmix64(seed & 0xFFFFFFFFFFFFFFFF, count, _ptr(out))
    return out


def random_matrix(n: int, dtype=np.float64, seed: int = 0, lo: float = -0.5,
                  hi: float = 0.5) -> np.ndarray:
    """linalg.py:127-148, returned as a plain C-contiguous ndarray."""
    if n < 1:
        raise ValueError(f"matrix order must be >= 1, got {n}")
    if not lo < hi:
        raise ValueError(f"need lo < hi, got [{lo}, {hi})")
    dtype = np.dtype(dtype)
    out = np.empty((n, n), dtype=dtype)
    fn = lib().mxo_random_f32 if dtype == np.float32 else lib().mxo_random_f64
    fn(n * n, seed & 0xFFFFFFFFFFFFFFFF, float(lo), float(hi), _ptr(out))
    return out


def scaled_input(n: int, dtype=np.float32, seed: int = 42) -> np.ndarray:
    """SURVEY §8(d) input recipe: fl_dtype(random_matrix(n, F64, seed) * sqrt(12/n)).

    Uniform[-1/2, 1/2) has variance 1/12, so the spectral radius is ~1 and
    every BASELINE power stays finite.
    """
    s = math.sqrt(12.0 / n)
    return (random_matrix(n, np.float64, seed) * s).astype(dtype)


def scaled_batch(n: int, batch: int, dtype=np.float32, seed0: int = 42,
                 indices=None) -> np.ndarray:
    """Batch element i uses seed seed0 + i."""
    idx = range(batch) if indices is None else indices
    return np.stack([scaled_input(n, dtype, seed0 + i) for i in idx])


# --- arithmetic --------------------------------------------------------------

def matmul(a: np.ndarray, b: np.ndarray, threads: int = 0) -> np.ndarray:
    """matmul_naive (linalg.py:151-164), bit-exact."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape and a.ndim == 2 and a.shape[0] == a.shape[1]
    assert a.dtype == b.dtype and a.dtype in (np.float32, np.float64)
    c = np.empty_like(a)
    fn = lib().mxo_matmul_f32 if a.dtype == np.float32 else lib().mxo_matmul_f64
    fn(a.shape[0], _ptr(a), _ptr(b), _ptr(c), threads or max_threads())
    return c


def matmul_rows(a: np.ndarray, b: np.ndarray, r0: int, r1: int, threads: int = 0) -> np.ndarray:
    """Rows [r0, r1) of matmul_naive(a, b) — a bounded sample of one multiply."""
    n = a.shape[0]
    c = np.empty((r1 - r0, n), dtype=a.dtype)
    fn = lib().mxo_matmul_rows_f32 if a.dtype == np.float32 else lib().mxo_matmul_rows_f64
    fn(n, r0, r1, _ptr(a), _ptr(b), _ptr(c), threads or max_threads())
    return c


def plan(power: int) -> str:
    """plan_exponentiation (expo.py:60-75) as a string of 'S'/'M'."""
    if power < 0:
        raise ValueError(f"power must be >= 0, got {power}")
    buf = ctypes.create_string_buffer(256)
    m = lib().mxo_plan(power, buf, 256)
    return buf.raw[:m].decode()


def multiply_count(power: int) -> int:
    return power.bit_length() - 1 + bin(power).count("1") - 1 if power >= 1 else 0


def exponentiate(a: np.ndarray, power: int, threads: int = 0) -> np.ndarray:
    """exponentiate(a, power, naive_backend()) (expo.py:121-139), bit-exact."""
    a = np.ascontiguousarray(a)
    if power < 0:
        raise ValueError(f"power must be >= 0, got {power}")
    out = np.empty_like(a)
    fn = lib().mxo_exponentiate_f32 if a.dtype == np.float32 else lib().mxo_exponentiate_f64
    fn(a.shape[0], power, _ptr(a), _ptr(out), threads or max_threads())
    return out


def exponentiate_batched(a: np.ndarray, power: int, threads: int = 0) -> np.ndarray:
    """Independent float32 chains over a (batch, n, n) stack."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty_like(a)
    lib().mxo_exponentiate_batched_f32(a.shape[1], a.shape[0], power, _ptr(a), _ptr(out),
                                       threads or max_threads())
    return out


def matmul_mod(a: np.ndarray, b: np.ndarray, p: int, threads: int = 0) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    c = np.empty_like(a)
    lib().mxo_matmul_mod(a.shape[0], p, _ptr(a), _ptr(b), _ptr(c), threads or max_threads())
    return c


def exponentiate_mod(a: np.ndarray, power: int, p: int, threads: int = 0) -> np.ndarray:
    """A^power mod p, exact (plan semantics of expo.py:121-139)."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    out = np.empty_like(a)
    lib().mxo_exponentiate_mod(a.shape[0], power, p, _ptr(a), _ptr(out),
                               threads or max_threads())
    return out


# --- metrics / tolerances -----------------------------------------------------

def compare(result: np.ndarray, reference: np.ndarray):
    """(max_abs, max_rel, frobenius_rel) in f64 — linalg.py:209-232."""
    res = np.asarray(result, dtype=np.float64)
    ref = np.asarray(reference, dtype=np.float64)
    diff = np.abs(res - ref)
    max_abs = float(diff.max())
    denom = float(np.abs(ref).max())
    if denom == 0.0:
        max_rel = 0.0 if max_abs == 0.0 else math.inf
    else:
        max_rel = max_abs / denom
    fro_ref = float(np.sqrt(np.sum(ref * ref)))
    fro_diff = float(np.sqrt(np.sum(diff * diff)))
    if fro_ref == 0.0:
        fro = 0.0 if fro_diff == 0.0 else math.inf
    else:
        fro = fro_diff / fro_ref
    return max_abs, max_rel, fro


def _u(dtype) -> float:
    return U32 if np.dtype(dtype) == np.float32 else U64


def oracle_tol(power: int, n: int, dtype) -> float:
    """tolerances.py:311-313: power * n * u * 64 (max_rel)."""
    return power * n * _u(dtype) * 64


def device_tol(n: int, dtype) -> float:
    """tolerances.py:316-319: n * u * 64 (max_rel, per multiply)."""
    return n * _u(dtype) * 64


def fro_tol(n: int, power: int, dtype) -> float:
    """relative Frobenius tolerance 16 * m(k) * sqrt(n) * u.

    m(k) = floor(log2 k) + popcount(k) - 1 is the multiply count (~log2 k), so
    the bound scales with log2 k as BASELINE.json's north_star requires.
    """
    return 16 * max(multiply_count(power), 1) * math.sqrt(n) * _u(dtype)
