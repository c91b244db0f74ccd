"""Matrix power plans and execution (mirrors matexpo/expo.py).

Same names, argument meaning and error behaviour as the reference:

* ``plan_exponentiation`` (expo.py:60-75): left-to-right binary plan.
* ``Backend`` / ``CountingBackend`` (expo.py:78-109): the multiply plugin.
* ``exponentiate(a, power, backend)`` (expo.py:121-139): A^0 = I, A^1 is
  ``a`` itself with zero multiplies, otherwise exactly
  floor(log2 N) + popcount(N) - 1 ``backend.multiply`` calls, the
  accumulator on the left, failures wrapped as ``BackendStepError``.
* ``repeated_exponentiate`` (expo.py:142-156), ``count_transfers``
  (expo.py:159-169), ``multiply_count_for`` (expo.py:172-180).

What is new is ``b200_backend()``: a ``Backend`` whose ``multiply`` is one
sm_100a tensor-core GEMM, and which ``exponentiate`` recognises so that the
whole chain runs as ONE C-ABI call (one upload, a CUDA-graph replay of the
plan over HBM ping-pong buffers, one readback) — the device chain of
gpuExponentiate (gpu-backend/src/host.ts:106-141).  Passing it to the
reference's own ``matexpo.exponentiate`` also works (per-multiply path).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .errors import BackendStepError, UnsupportedPowerError
from .linalg import Matrix, as_array, check_pair, identity, wrap_like
from .dtypes import DType


class Step(enum.Enum):
    SQUARE = "S"
    MULTIPLY_BASE = "M"


class Strategy(enum.Enum):
    REPEATED = "repeated"
    SQUARED = "squared"

    @classmethod
    def parse(cls, name: str) -> "Strategy":
        try:
            return cls(name.lower())
        except ValueError:
            raise ValueError(
                f"unknown strategy {name!r}; expected one of: repeated, squared"
            ) from None


@dataclass(frozen=True)
class ExponentPlan:
    """Left-to-right binary plan for A**power (expo.py:39-57)."""

    power: int
    steps: tuple

    @property
    def multiply_count(self) -> int:
        return len(self.steps)

    @property
    def square_count(self) -> int:
        return sum(1 for s in self.steps if s is Step.SQUARE)

    def as_string(self) -> str:
        return "".join(s.value for s in self.steps)


def plan_exponentiation(power: int) -> ExponentPlan:
    """Scan the bits of ``power`` below the leading one, high to low: one
    SQUARE per bit, then MULTIPLY_BASE when the bit is set."""
    if power < 0:
        raise ValueError(f"power must be >= 0, got {power}")
    steps = []
    for shift in reversed(range(max(power.bit_length() - 1, 0))):
        steps.append(Step.SQUARE)
        if (power >> shift) & 1:
            steps.append(Step.MULTIPLY_BASE)
    return ExponentPlan(power, tuple(steps))


def count_transfers(plan: ExponentPlan, strategy: Strategy) -> int:
    """Modeled host<->device transfers: REPEATED moves one matrix per power
    step; SQUARED uploads once and reads back once (expo.py:159-169)."""
    return plan.power if strategy is Strategy.REPEATED else 2


def multiply_count_for(strategy: Strategy, power: int) -> int:
    if strategy is Strategy.REPEATED:
        if power < 1:
            raise UnsupportedPowerError(f"repeated baseline needs power >= 1, got {power}")
        return power - 1
    return plan_exponentiation(power).multiply_count


@dataclass(frozen=True)
class Backend:
    """A named multiply routine plus its host-device transfer model."""

    name: str
    multiply: Callable
    transfer_cost_model: Callable = field(
        default=lambda plan, strategy: count_transfers(plan, strategy)
    )


class CountingBackend:
    """Wrap a backend and count multiply invocations (expo.py:89-109)."""

    def __init__(self, inner):
        self.inner = inner
        self.calls = 0

    @property
    def name(self) -> str:
        return self.inner.name

    @property
    def transfer_cost_model(self):
        return self.inner.transfer_cost_model

    def multiply(self, a, b):
        self.calls += 1
        return self.inner.multiply(a, b)

    def reset(self) -> None:
        self.calls = 0


class B200Backend(Backend):
    """Marker subclass: ``exponentiate`` runs the whole plan on the device."""

    @property
    def engine(self):
        from .engine import default_engine

        return default_engine(self.device)

    device: int = 0


def b200_backend(device: int = 0) -> Backend:
    """The sm_100a tensor-core backend (3xTF32 for f32, DMMA for f64)."""
    from .engine import default_engine

    def multiply(a, b):
        check_pair(a, b)
        out = default_engine(device).multiply(as_array(a), as_array(b))
        return wrap_like(a, out)

    be = B200Backend("b200", multiply)
    object.__setattr__(be, "device", device)
    return be


def exponentiate(a, power: int, backend=None):
    """A**power by square-and-multiply; A**0 is the identity.

    With a B200 backend (or ``backend=None``) the whole plan runs on the
    device in one call; any other backend is driven step by step exactly as
    the reference does, invoking ``backend.multiply`` once per plan step.
    """
    plan = plan_exponentiation(power)
    if power == 0:
        arr = as_array(a)
        return wrap_like(a, identity(arr.shape[0], DType.of(arr)).array.copy())
    if power == 1:
        return a
    if backend is None or isinstance(backend, B200Backend):
        device = getattr(backend, "device", 0) if backend is not None else 0
        from .engine import default_engine

        arr = np.ascontiguousarray(as_array(a))
        out = default_engine(device).power(arr, power)
        return wrap_like(a, out)
    acc = a
    for index, step in enumerate(plan.steps):
        try:
            acc = backend.multiply(acc, acc) if step is Step.SQUARE else backend.multiply(acc, a)
        except Exception as exc:  # noqa: BLE001 - annotate and re-raise
            raise BackendStepError(index, step.name, exc) from exc
    return acc


def exponentiate_batched(a: np.ndarray, power: int, device: int = 0,
                         out: np.ndarray | None = None) -> np.ndarray:
    """A_i**power for a (batch, n, n) float32/float64 stack (BASELINE config 3).
    ``out`` (optional): a C-contiguous array of a's shape and dtype to write
    into — reusing it spares the first-touch page faults of a fresh result."""
    if power < 0:
        raise ValueError(f"power must be >= 0, got {power}")
    from .engine import default_engine

    return default_engine(device).power_batched(np.ascontiguousarray(a), power, out=out)


def exponentiate_multi(a, power: int, devices=None) -> np.ndarray:
    """A**power on several GPUs of this process (the C ABI's mxp_power_multi):
    a (batch, n, n) stack is sharded by matrices, one n x n FP32 matrix by
    rows with the exchange fused into the GEMM epilogue.  ``a`` may be a
    Matrix or an ndarray; the result is an ndarray.  The reference has no
    multi-device path; the plan, k = 0 / 1 and error semantics
    are exponentiate's."""
    if power < 0:
        raise ValueError(f"power must be >= 0, got {power}")
    from .engine import power_multi

    arr = a.array if hasattr(a, "array") else a
    return power_multi(np.ascontiguousarray(arr), power, devices)


def repeated_exponentiate(a, power: int, backend):
    """A**power by power-1 successive multiplies (expo.py:142-156)."""
    if power < 1:
        raise UnsupportedPowerError(f"repeated baseline needs power >= 1, got {power}")
    acc = a
    for index in range(power - 1):
        try:
            acc = backend.multiply(acc, a)
        except Exception as exc:  # noqa: BLE001
            raise BackendStepError(index, "MULTIPLY_BASE", exc) from exc
    return acc
