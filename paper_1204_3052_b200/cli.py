"""Command line (mirrors matexpo/cli.py:73-237 for the b200 backend):

    python -m paper_1204_3052_b200.cli verify --size 512 --power 1000 [--dtype f32]
    python -m paper_1204_3052_b200.cli bench --sizes 128,512 --powers 64,1000 --csv -

Exit codes as the reference (cli.py:217-233): 0 ok, 1 validation error,
2 runtime failure, 3 verify FAIL.  `verify` compares against the F64
repeated-multiply oracle computed on the device with the
reference's `oracle_tol` (max_rel) and additionally reports the relative
Frobenius error against `fro_tol`.
"""

from __future__ import annotations

import argparse
import sys
from typing import Optional, Sequence

import numpy as np


def _int_list(text: str):
    return [int(t) for t in text.split(",") if t]


def _str_list(text: str):
    return [t for t in text.split(",") if t]


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="matexpo-b200",
                                     description="B200 matrix exponentiation")
    sub = parser.add_subparsers(dest="command", required=True)
    bench = sub.add_parser("bench", help="sweep sizes x powers x strategies")
    bench.add_argument("--sizes", type=_int_list, required=True)
    bench.add_argument("--powers", type=_int_list, required=True)
    bench.add_argument("--strategies", type=_str_list, default=["repeated", "squared"])
    bench.add_argument("--backend", dest="backends", type=_str_list, default=["b200"])
    bench.add_argument("--dtype", default="f32", choices=("f32", "f64"))
    bench.add_argument("--seed", type=int, default=42)
    bench.add_argument("--reps", type=int, default=5)
    bench.add_argument("--no-oracle", action="store_true")
    bench.add_argument("--extended", action="store_true", help="append the B200 CSV columns")
    bench.add_argument("--csv", default="-", help="CSV output path, or - for stdout")
    bench.add_argument("--table", help="the paper's comparison table: output path, or - for stdout")
    bench.add_argument("--baseline-csv", help="CSV with the reference's naive (sequential CPU) "
                       "rows for --table, written by the reference CLI")
    bench.set_defaults(func=cmd_bench)
    verify = sub.add_parser("verify", help="oracle comparison for one grid point")
    verify.add_argument("--size", type=int, required=True)
    verify.add_argument("--power", type=int, required=True)
    verify.add_argument("--strategy", default="squared", choices=("repeated", "squared"))
    verify.add_argument("--backend", default="b200", choices=("b200",))
    verify.add_argument("--dtype", default="f64", choices=("f32", "f64"))
    verify.add_argument("--seed", type=int, default=42)
    verify.add_argument("--scaled", action="store_true",
                        help="spectrally normalised input (SURVEY §8(d)) instead of U[-1/2,1/2)")
    verify.set_defaults(func=cmd_verify)
    return parser


def cmd_bench(args) -> int:
    from . import harness
    from .dtypes import DType
    from .expo import Strategy

    cfg = harness.BenchConfig(sizes=args.sizes, powers=args.powers,
                              strategies=[Strategy.parse(s) for s in args.strategies],
                              backends=args.backends, dtype=DType.parse(args.dtype),
                              seed=args.seed, repetitions=args.reps, oracle=not args.no_oracle)
    if args.table and not args.baseline_csv:
        raise ValueError("--table needs --baseline-csv (the reference's naive rows)")
    records = harness.run_benchmark(cfg)
    if args.csv == "-":
        if not args.table:
            harness.emit_csv(records, sys.stdout, args.extended)
    else:
        harness.emit_csv(records, args.csv, args.extended)
    if args.table:
        base = [r for r in harness.read_csv(args.baseline_csv) if r.backend == "naive"]
        texts = [harness.emit_table([r for r in records + base if r.size == size])
                 for size in sorted({r.size for r in records})]
        text = "\n".join(texts)
        if args.table == "-":
            sys.stdout.write(text)
        else:
            with open(args.table, "w", encoding="utf-8") as fh:
                fh.write(text)
    return 0


def cmd_verify(args) -> int:
    from . import harness
    from .dtypes import DType
    from .expo import Strategy, exponentiate, repeated_exponentiate
    from .generate import random_matrix, scaled_input
    from .linalg import compare
    from .tolerances import fro_tol, oracle_tol

    dtype = DType.parse(args.dtype)
    base = (scaled_input(args.size, dtype, args.seed) if args.scaled
            else random_matrix(args.size, dtype, args.seed))
    backend = harness.make_backend(args.backend)
    strategy = Strategy.parse(args.strategy)
    if strategy is Strategy.REPEATED:
        result = repeated_exponentiate(base, args.power, backend)
    else:
        result = exponentiate(base, args.power, backend)
    oracle = harness.device_oracle(base, args.power)
    metrics = compare(result.array.astype(np.float64), oracle)
    tol = oracle_tol(args.power, args.size, dtype)
    ok = metrics.max_rel <= tol
    print(f"size={args.size}")
    print(f"power={args.power}")
    print(f"strategy={strategy.value}")
    print(f"backend={backend.name}")
    print(f"max_abs_err={metrics.max_abs!r}")
    print(f"max_rel_err={metrics.max_rel!r}")
    print(f"tolerance={tol!r}")
    print(f"frobenius_rel_err={metrics.frobenius_rel!r}")
    print(f"frobenius_tolerance={fro_tol(args.size, args.power, dtype)!r}")
    print(f"verdict={'PASS' if ok else 'FAIL'}")
    return 0 if ok else 3


def main(argv: Optional[Sequence[str]] = None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code in (0, None) else 1
    try:
        return args.func(args)
    except BrokenPipeError:
        return 0
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except Exception as exc:  # noqa: BLE001 - CLI boundary
        print(f"runtime failure: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
