"""Host-side mirror of the reference API (no GPU): plan, backend plugin,
exponentiate driving a generic backend, errors, Matrix, compare, tolerances.
Mirrors pkg/tests/test_expo.py / test_linalg.py for the names this package keeps."""

import math
import os

import numpy as np
import pytest
from hypothesis import given, strategies as st

import oracle
import paper_1204_3052_b200 as mx
from paper_1204_3052_b200 import (
    Backend,
    BackendStepError,
    CountingBackend,
    DType,
    Matrix,
    Step,
    Strategy,
    UnsupportedPowerError,
    count_transfers,
    exponentiate,
    multiply_count_for,
    plan_exponentiation,
    repeated_exponentiate,
)


def stub():
    return CountingBackend(Backend("stub", lambda a, b: a))


def oracle_backend():
    """The CPU oracle as a backend — test infrastructure only."""
    return Backend("oracle", lambda a, b: Matrix(oracle.matmul(a.array, b.array), copy=False))


def law(p):
    return p.bit_length() - 1 + bin(p).count("1") - 1 if p >= 1 else 0


def test_small_plans():
    assert plan_exponentiation(0).steps == ()
    assert plan_exponentiation(1).steps == ()
    assert plan_exponentiation(2).steps == (Step.SQUARE,)
    assert plan_exponentiation(3).steps == (Step.SQUARE, Step.MULTIPLY_BASE)
    assert plan_exponentiation(13).as_string() == "SMSSM"
    assert plan_exponentiation(1024).square_count == 10
    assert plan_exponentiation(1023).square_count == 9
    with pytest.raises(ValueError):
        plan_exponentiation(-1)


@given(power=st.integers(1, 2**20))
def test_count_law(power):
    assert plan_exponentiation(power).multiply_count == law(power)
    assert plan_exponentiation(power).as_string() == oracle.plan(power)


@given(power=st.integers(1, 2**16))
def test_plan_executes_to_the_power(power):
    e = 1
    for s in plan_exponentiation(power).steps:
        e = e * 2 if s is Step.SQUARE else e + 1
    assert e == power


def test_invocations_match_plan_with_generic_backend():
    a = Matrix(np.eye(2))
    for power in (1, 13, 512, 1024, 4096):
        be = stub()
        exponentiate(a, power, be)
        assert be.calls == law(power)


def test_power_zero_one_semantics():
    a = Matrix(oracle.random_matrix(4, np.float32, 3))
    be = stub()
    assert exponentiate(a, 1, be) is a and be.calls == 0
    out = exponentiate(a, 0, be)
    assert np.array_equal(out.array, np.eye(4)) and out.dtype is DType.F32


def test_step_failure_is_annotated():
    boom = RuntimeError("device fell over")
    calls = []

    def flaky(a, b):
        calls.append(1)
        if len(calls) == 2:
            raise boom
        return a

    with pytest.raises(BackendStepError) as ei:
        exponentiate(Matrix(np.eye(2)), 8, Backend("flaky", flaky))
    assert ei.value.step_index == 1 and ei.value.step_name == "SQUARE"
    assert ei.value.__cause__ is boom


def test_generic_backend_chain_bitwise_equals_oracle(golden):
    arrays, _ = golden
    for n in (4, 16):
        a = Matrix(arrays[f"in_{n}_f32"])
        for k in (2, 7, 13, 64):
            got = exponentiate(a, k, oracle_backend())
            assert got.array.tobytes() == arrays[f"exp_{n}_f32_{k}"].tobytes()


def test_repeated_and_strategy():
    assert multiply_count_for(Strategy.REPEATED, 512) == 511
    assert multiply_count_for(Strategy.SQUARED, 512) == 9
    with pytest.raises(UnsupportedPowerError):
        multiply_count_for(Strategy.REPEATED, 0)
    with pytest.raises(UnsupportedPowerError):
        repeated_exponentiate(Matrix(np.eye(2)), 0, stub())
    be = stub()
    repeated_exponentiate(Matrix(np.eye(2)), 64, be)
    assert be.calls == 63
    assert Strategy.parse("SQUARED") is Strategy.SQUARED
    for p in (1, 2, 13, 1024):
        assert count_transfers(plan_exponentiation(p), Strategy.SQUARED) == 2
        assert count_transfers(plan_exponentiation(p), Strategy.REPEATED) == p
    assert mx.b200_backend().transfer_cost_model(plan_exponentiation(1024), Strategy.SQUARED) == 2


def test_matrix_contract():
    arr = np.zeros((3, 3))
    m = Matrix(arr)
    arr[0, 0] = 7
    assert m.array[0, 0] == 0
    with pytest.raises(ValueError):
        m.array[0, 0] = 1
    with pytest.raises(mx.ShapeError):
        Matrix(np.zeros((2, 3)))
    with pytest.raises(mx.ShapeError):
        Matrix(np.zeros((2, 2), dtype=np.int64))
    with pytest.raises(mx.InvalidDimensionError):
        mx.identity(0)
    assert Matrix.from_rows([[1, 2], [3, 4]], DType.F32).data.tolist() == [1, 2, 3, 4]


def test_compare_semantics():
    z = mx.zeros(2)
    assert tuple(mx.compare(z, z)) == (0.0, 0.0, 0.0)
    off = Matrix.from_rows([[0.0, 1.0], [0.0, 0.0]])
    m = mx.compare(off, z)
    assert m.max_abs == 1.0 and m.max_rel == math.inf and m.frobenius_rel == math.inf
    ref = Matrix.from_rows([[2.0, 0.0], [0.0, 2.0]])
    res = Matrix.from_rows([[2.0, 0.0], [0.0, 2.5]])
    assert mx.compare(res, ref).max_rel == 0.25


def test_tolerances_match_reference_and_survey():
    assert mx.oracle_tol(1024, 8192, DType.F32) == 1024 * 8192 * 2**-24 * 64
    assert mx.device_tol(64, DType.F32) == 64 * 2**-24 * 64
    # SURVEY §8(d) values
    assert abs(mx.fro_tol(64, 16, DType.F32) - 3.1e-5) < 0.1e-5
    assert abs(mx.fro_tol(512, 1000, DType.F32) - 3.0e-4) < 0.1e-4
    assert abs(mx.fro_tol(128, 64, DType.F32) - 6.5e-5) < 0.1e-5
    assert abs(mx.fro_tol(8192, 1024, DType.F32) - 8.6e-4) < 0.1e-4


def test_wrap_like_reference_matrix_type():
    """Results come back in the caller's matrix class (reference interop)."""
    from paper_1204_3052_b200.linalg import wrap_like

    class Foreign:
        def __init__(self, array, copy=True):
            self.array = np.array(array)

    out = wrap_like(Foreign(np.eye(2)), np.ones((2, 2)))
    assert isinstance(out, Foreign)


# ------------------------------------------------------------------ text format (linalg.py:235-276)
UNIFORM_F32_SEED7_TEXT = (  # gpu-backend/test/helpers.ts:51-56 (independent producer)
    "4 f32\n"
    "-0.11017025 -0.4832117 0.40076068 0.0829303\n"
    "-0.047558106 -0.25056848 -0.032046996 -0.17192326\n"
    "-0.3657417 -0.0868586 -0.39644006 0.45987406\n"
    "0.4180196 0.37133175 0.36400765 0.048287418\n")


def test_text_format_matches_reference_fixture():
    import io

    m = Matrix(oracle.random_matrix(4, np.float32, 7))
    buf = io.StringIO()
    mx.write_matrix(m, buf)
    assert buf.getvalue() == UNIFORM_F32_SEED7_TEXT
    back = mx.read_matrix(io.StringIO(UNIFORM_F32_SEED7_TEXT))
    assert back.array.tobytes() == m.array.tobytes()


@given(seed=st.integers(0, 2**20), n=st.integers(1, 8), f64=st.booleans())
def test_text_round_trip_bitwise(seed, n, f64):
    import io

    m = Matrix(oracle.random_matrix(n, np.float64 if f64 else np.float32, seed, -100.0, 100.0))
    buf = io.StringIO()
    mx.write_matrix(m, buf)
    back = mx.read_matrix(io.StringIO(buf.getvalue()))
    assert back.array.tobytes() == m.array.tobytes()


def test_text_format_malformed():
    import io

    with pytest.raises(mx.ShapeError):
        mx.read_matrix(io.StringIO("2\n1 2\n3 4\n"))
    with pytest.raises(ValueError):
        mx.read_matrix(io.StringIO("2 f16\n1 2\n3 4\n"))
    with pytest.raises(mx.ShapeError):
        mx.read_matrix(io.StringIO("2 f64\n1 2 3\n4 5 6\n"))
    with pytest.raises(mx.InvalidDimensionError):
        mx.read_matrix(io.StringIO("0 f64\n"))


# ------------------------------------------------------------------ harness CSV (bench.py:259-305)
def test_csv_schema_is_the_reference_one():
    import io

    from paper_1204_3052_b200 import harness

    assert harness.CSV_HEADER == ("size,power,strategy,backend,seconds,multiply_count,"
                                  "transfer_count,max_rel_err,nonfinite")
    recs = [harness.BenchmarkRecord(64, 16, Strategy.SQUARED, "b200", 1.5e-5, 4, 2, 3e-7, False,
                                    1, "f32-3xtf32", 0.01, 0.1),
            harness.BenchmarkRecord(64, 16, Strategy.REPEATED, "b200", 2e-4, 15, 16, None, True)]
    for ext in (False, True):
        buf = io.StringIO()
        harness.emit_csv(recs, buf, extended=ext)
        back = harness.read_csv(io.StringIO(buf.getvalue()))
        assert [(r.power, r.strategy, r.max_rel_err, r.nonfinite) for r in back] == \
            [(16, Strategy.REPEATED, None, True), (16, Strategy.SQUARED, 3e-7, False)]
    with pytest.raises(mx.ConfigError):
        harness.make_backend("naive")
    with pytest.raises(mx.ConfigError):
        harness.validate_config(harness.BenchConfig(sizes=[0], powers=[-1]))


def test_cli_validation_exit_code():
    from paper_1204_3052_b200 import cli

    assert cli.main(["verify", "--size", "4"]) == 1  # missing --power: usage error -> 1
    assert cli.main(["bench", "--sizes", "4", "--powers", "2", "--backend", "naive"]) == 1


# ------------------------------------------------------------------ the paper's table (bench.py:330-395)
def test_emit_table_matches_the_reference_rendering():
    """tests/golden/table_expected.txt is the reference's own emit_table output
    for the records in table_records.csv (tests/golden/make_golden_table.py)."""
    from paper_1204_3052_b200 import harness

    here = os.path.join(os.path.dirname(__file__), "golden")
    recs = harness.read_csv(os.path.join(here, "table_records.csv"))
    with open(os.path.join(here, "table_expected.txt"), encoding="utf-8") as fh:
        assert harness.emit_table(recs) == fh.read()
    with pytest.raises(mx.TableError):
        harness.emit_table([r for r in recs if not (r.backend == "naive" and r.power == 16)])
    with pytest.raises(mx.TableError):
        harness.emit_table([])


def test_public_names_cover_the_reference_hot_path_surface():
    """Every name of the reference's __all__ (matexpo/__init__.py:93-166)
    that belongs to the hot path (SURVEY §2 ★) or its harness (§8(f1)) is
    public here too.  The rest is out of scope by design: the OpenCL tile
    menu (tiles.py), the work-group simulator (kernelsim.py), plots, and the
    CPU products naive/tiled (no CPU path in the product)."""
    import paper_1204_3052_b200 as mx

    out_of_scope = {
        "CoalescingReport", "DEFAULT_LOCAL_MEM_BUDGET", "LaunchError", "LaunchGeometry",
        "LocalMemoryError", "PlotError", "REVERSED", "ROW_MAJOR", "RaceVerdict", "Schedule",
        "TILE_MENU", "TileConfig", "TilingError", "TrafficReport", "UNROLL_FACTORS",
        "VECTOR_WIDTHS", "analyze_coalescing", "check_budget", "check_divisibility",
        "default_schedules", "detect_barrier_race", "emit_plot", "matmul_naive", "matmul_tiled",
        "naive_backend", "predict_traffic", "shuffle_schedule", "simulate_naive_matmul",
        "simulate_tiled_matmul", "staged_footprint_bytes", "tiled_backend",
        "unblocked_global_loads",
    }
    try:
        import importlib
        import sys

        sys.path.insert(0, "/root/reference/pkg/src")
        ref = importlib.import_module("matexpo")
        ref_all = set(ref.__all__)
    except ImportError:
        pytest.skip("reference not present (GPU box)")
    finally:
        if "/root/reference/pkg/src" in sys.path:
            sys.path.remove("/root/reference/pkg/src")
    missing = ref_all - set(mx.__all__) - out_of_scope
    assert not missing, sorted(missing)
    for name in ref_all - out_of_scope:
        assert getattr(mx, name) is not None, name
