"""Benchmark harness and backend registry, mirroring
matexpo/bench.py: `make_backend` (bench.py:53-66), `BenchConfig`
(bench.py:69-80), `BenchmarkRecord` + the CSV schema (bench.py:42, :83-98,
:259-305) and `run_benchmark` (bench.py:183-256) — with the B200 engine as
the backend and the oracle column computed on the device (F64 repeated
multiplies), so `oracle_cap` no longer limits sizes.

CSV: `emit_csv(..., extended=False)` writes exactly the reference's 9-column
schema (readable by the reference's own `read_csv`); `extended=True` appends
`gpus,dtype_mode,device_ms,tflops`.
"""

from __future__ import annotations

import statistics
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence, TextIO, Union

import numpy as np

from .dtypes import DType
from .errors import ConfigError, TableError
from .expo import (
    Backend,
    CountingBackend,
    Strategy,
    b200_backend,
    count_transfers,
    exponentiate,
    plan_exponentiation,
    repeated_exponentiate,
)
from .generate import random_matrix
from .linalg import Matrix, compare

BACKEND_NAMES = ("b200",)
CSV_HEADER = ("size,power,strategy,backend,seconds,multiply_count,transfer_count,max_rel_err,"
              "nonfinite")
CSV_EXTRA = "gpus,dtype_mode,device_ms,tflops"
# the paper's comparison table (bench.py:44-50 of the reference)
TABLE_ROW_LABELS = (
    "Naïve GPU (In Sec)",
    "Sequential CPU (In Sec)",
    "Naïve Speed UP",
    "Our Approach (In Sec)",
    "Our Approach vs Naïve GPU",
)


def make_backend(name: str, tile=None) -> Backend:
    """Registered backends by name (bench.py:53-66); `tile` is accepted for
    signature compatibility and ignored (tcgen05 tiling is not user-chosen)."""
    if name == "b200":
        return b200_backend()
    raise ConfigError(f"unknown backend {name!r}; expected one of {BACKEND_NAMES}")


@dataclass
class BenchConfig:
    sizes: Sequence[int]
    powers: Sequence[int]
    strategies: Sequence[Strategy] = (Strategy.REPEATED, Strategy.SQUARED)
    backends: Sequence[str] = ("b200",)
    dtype: DType = DType.F32
    seed: int = 42
    repetitions: int = 5
    oracle: bool = True


@dataclass(frozen=True)
class BenchmarkRecord:
    size: int
    power: int
    strategy: Strategy
    backend: str
    seconds: float
    multiply_count: int
    transfer_count: int
    max_rel_err: Optional[float]
    nonfinite: bool
    gpus: int = 1
    dtype_mode: str = "f32-3xtf32"
    device_ms: Optional[float] = None
    tflops: Optional[float] = None

    def sort_key(self):
        return (self.size, self.power, self.strategy.value, self.backend)


def validate_config(config: BenchConfig) -> None:
    problems = []
    if not config.sizes:
        problems.append("sizes must be non-empty")
    if not config.powers:
        problems.append("powers must be non-empty")
    if not config.strategies:
        problems.append("strategies must be non-empty")
    for n in config.sizes:
        if n < 1:
            problems.append(f"size {n} must be >= 1")
    for p in config.powers:
        if p < 1:
            problems.append(f"power {p} must be >= 1")
    if config.repetitions < 1:
        problems.append("repetitions must be >= 1")
    for name in config.backends:
        if name not in BACKEND_NAMES:
            problems.append(f"unknown backend {name!r}; expected one of {BACKEND_NAMES}")
    if problems:
        raise ConfigError("; ".join(problems))


def device_oracle(base: Matrix, power: int) -> np.ndarray:
    """F64 repeated-multiply oracle (bench.py:178-180) on the device."""
    from .engine import default_engine

    return default_engine().repeated_power(base.array.astype(np.float64), power)


def run_benchmark(config: BenchConfig) -> list:
    validate_config(config)
    records = []
    for size in config.sizes:
        base = random_matrix(size, config.dtype, config.seed)
        for power in config.powers:
            ref = device_oracle(base, power) if config.oracle else None
            for strategy in config.strategies:
                for name in config.backends:
                    records.append(_run_point(config, base, size, power, strategy, name, ref))
    return records


def _run_point(config, base, size, power, strategy, name, ref):
    from .engine import default_engine

    backend = make_backend(name)
    counting = CountingBackend(backend)
    if strategy is Strategy.REPEATED:
        run = lambda: repeated_exponentiate(base, power, counting)  # noqa: E731
        result = run()
        count = counting.calls
    else:
        run = lambda: exponentiate(base, power, backend)  # noqa: E731
        result = run()
        count = plan_exponentiation(power).multiply_count
    samples = []
    for _ in range(config.repetitions):
        t0 = time.perf_counter()
        run()
        samples.append(time.perf_counter() - t0)
    seconds = statistics.median(samples)
    dev_ms = default_engine().last_stats.device_ms if strategy is Strategy.SQUARED else None
    transfers = backend.transfer_cost_model(plan_exponentiation(power), strategy)
    arr = result.array
    nonfinite = not bool(np.isfinite(arr).all())
    err = None
    if ref is not None:
        err = compare(arr.astype(np.float64), ref).max_rel
    flops = 2.0 * size ** 3 * count
    return BenchmarkRecord(size, power, strategy, backend.name, seconds, count, transfers, err,
                           nonfinite, 1, "f32-3xtf32" if config.dtype is DType.F32 else "f64-dmma",
                           dev_ms, flops / seconds / 1e12)


def emit_csv(records, dest: Union[str, TextIO], extended: bool = False) -> None:
    if hasattr(dest, "write"):
        _write_csv(records, dest, extended)
    else:
        with open(dest, "w", encoding="utf-8") as fh:
            _write_csv(records, fh, extended)


def _write_csv(records, fh: TextIO, extended: bool) -> None:
    fh.write(CSV_HEADER + ("," + CSV_EXTRA if extended else "") + "\n")
    for r in sorted(records, key=BenchmarkRecord.sort_key):
        err = "" if r.max_rel_err is None else repr(float(r.max_rel_err))
        line = (f"{r.size},{r.power},{r.strategy.value},{r.backend},{r.seconds!r},"
                f"{r.multiply_count},{r.transfer_count},{err},{'true' if r.nonfinite else 'false'}")
        if extended:
            dm = "" if r.device_ms is None else repr(float(r.device_ms))
            tf = "" if r.tflops is None else repr(float(r.tflops))
            line += f",{r.gpus},{r.dtype_mode},{dm},{tf}"
        fh.write(line + "\n")


def read_csv(src: Union[str, TextIO]) -> list:
    if hasattr(src, "read"):
        return _read_csv(src)
    with open(src, "r", encoding="utf-8") as fh:
        return _read_csv(fh)


def _read_csv(fh: TextIO) -> list:
    header = fh.readline().strip()
    extended = header == CSV_HEADER + "," + CSV_EXTRA
    if header != CSV_HEADER and not extended:
        raise ValueError(f"unexpected CSV header {header!r}")
    out = []
    for line in fh:
        line = line.rstrip("\n")
        if not line:
            continue
        p = line.split(",")
        if len(p) != (13 if extended else 9):
            raise ValueError(f"malformed CSV row {line!r}")
        rec = dict(size=int(p[0]), power=int(p[1]), strategy=Strategy.parse(p[2]), backend=p[3],
                   seconds=float(p[4]), multiply_count=int(p[5]), transfer_count=int(p[6]),
                   max_rel_err=None if p[7] == "" else float(p[7]), nonfinite=p[8] == "true")
        if extended:
            rec.update(gpus=int(p[9]), dtype_mode=p[10],
                       device_ms=None if p[11] == "" else float(p[11]),
                       tflops=None if p[12] == "" else float(p[12]))
        out.append(BenchmarkRecord(**rec))
    return out


# --------------------------------------------------------------------------- table
def emit_table(records) -> str:
    """The paper's five-row comparison table for one matrix size, in the
    reference's text format (bench.py:330-395): the sequential CPU row is
    REPEATED on the ``naive`` backend, "Naïve GPU" is REPEATED on the
    accelerated backend (here b200: k-1 device GEMMs) and "Our Approach" is
    SQUARED on it (the CUDA-graph chain); the two speed-up rows are time ratios
    with two decimals.  The naive rows are the reference's own measurements:
    read them from a CSV written by the reference CLI (``matexpo bench
    --backends naive --strategies repeated --csv ref.csv``) and pass the
    records of both files; a missing cell raises TableError."""
    from .expo import Strategy

    if not records:
        raise TableError("no records to tabulate")
    sizes = sorted({r.size for r in records})
    if len(sizes) != 1:
        raise TableError(f"records span sizes {sizes}; tabulate one size at a time")
    accel = sorted({r.backend for r in records if r.backend != "naive"})
    if not accel:
        raise TableError("need a non-naive backend for the accelerated rows")
    if len(accel) > 1:
        raise TableError(f"ambiguous accelerated backend: {accel}; filter records first")
    roles = {"seq": (Strategy.REPEATED, "naive"), "gpu": (Strategy.REPEATED, accel[0]),
             "ours": (Strategy.SQUARED, accel[0])}
    powers = sorted({r.power for r in records})
    cells = {role: {} for role in roles}
    for r in records:
        for role, (strategy, backend) in roles.items():
            if r.strategy is strategy and r.backend == backend:
                cells[role][r.power] = r.seconds
    missing = [f"{strategy.value}/{backend} @ power={p}" for role, (strategy, backend)
               in roles.items() for p in powers if p not in cells[role]]
    if missing:
        raise TableError("missing cells: " + ", ".join(missing))

    def secs(v):
        return f"{v:.6g}"

    def ratio(v):
        text = f"{v:.2f}"
        return text.rstrip("0").rstrip(".") if "." in text else text

    seq, gpu, ours = cells["seq"], cells["gpu"], cells["ours"]
    rows = [(TABLE_ROW_LABELS[0], [secs(gpu[p]) for p in powers]),
            (TABLE_ROW_LABELS[1], [secs(seq[p]) for p in powers]),
            (TABLE_ROW_LABELS[2], [ratio(seq[p] / gpu[p]) for p in powers]),
            (TABLE_ROW_LABELS[3], [secs(ours[p]) for p in powers]),
            (TABLE_ROW_LABELS[4], [ratio(gpu[p] / ours[p]) for p in powers])]
    lw = max(len(label) for label, _ in rows)
    widths = [max(len(str(p)), *(len(vals[i]) for _, vals in rows)) for i, p in enumerate(powers)]
    out = [f"Matrix size {sizes[0]} x {sizes[0]}",
           " " * lw + "  " + "  ".join(str(p).rjust(w) for p, w in zip(powers, widths))]
    out += [label.ljust(lw) + "  " + "  ".join(v.rjust(w) for v, w in zip(vals, widths))
            for label, vals in rows]
    return "\n".join(out) + "\n"
