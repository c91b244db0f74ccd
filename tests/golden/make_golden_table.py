"""Fixtures for the paper-table path (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_table.py

* table_records.csv / table_expected.txt: a fixed record set in the
  reference's CSV schema and the reference's own ``emit_table`` rendering of
  it (bench.py:330-395) — pins our harness.emit_table byte for byte.
* ref_naive_64.csv: the reference CLI's sequential-CPU rows (REPEATED on the
  naive backend, 64x64 f32, seed 42) for powers 2, 16, 64, measured on this
  container's CPU; `cli bench --table - --baseline-csv` merges them with the
  B200 rows (tests/test_gpu_parity.py).
"""

import os
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from matexpo.bench import BenchmarkRecord, emit_csv, emit_table  # noqa: E402
from matexpo.expo import Strategy  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    recs = []
    times = {("repeated", "naive"): (0.0123, 0.98765, 4.2),
             ("repeated", "b200"): (0.00031, 0.0051, 0.0203),
             ("squared", "b200"): (0.000101, 0.0001234567, 0.000130)}
    for (strategy, backend), secs in times.items():
        for power, s in zip((2, 16, 64), secs):
            mult = power - 1 if strategy == "repeated" else {2: 1, 16: 4, 64: 6}[power]
            recs.append(BenchmarkRecord(64, power, Strategy.parse(strategy), backend, s, mult,
                                        2 * mult + 1 if strategy == "repeated" else 2, 1e-7,
                                        False))
    emit_csv(recs, os.path.join(HERE, "table_records.csv"))
    with open(os.path.join(HERE, "table_expected.txt"), "w", encoding="utf-8") as fh:
        fh.write(emit_table(recs))
    from matexpo.cli import main as ref_cli

    rc = ref_cli(["bench", "--sizes", "64", "--powers", "2,16,64", "--strategies", "repeated",
                  "--backend", "naive", "--reps", "3", "--csv",
                  os.path.join(HERE, "ref_naive_64.csv")])
    assert rc == 0, rc


if __name__ == "__main__":
    main()
