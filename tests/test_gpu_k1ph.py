"""K1PH: single-matrix FP32 chains at the CTA-pair sizes on scaled fp16x2
planes (kernels_f16x2.cu), the 3xTF32 recomputation it falls back to when a
product loses dynamic range, and the per-handle datapath switch.

Parity: relative Frobenius error against the oracle within fro_tol (SURVEY
§8(d)), and no worse than the 3xTF32 chain's own error by more than a
rounding-level margin (the operand precision is the same 22 bits)."""

import numpy as np
import pytest

import oracle
import paper_1204_3052_b200 as mx

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    return mx.Engine(0)


def _both(eng, a, k):
    eng.set_f32_datapath("auto")
    g16 = eng.power(a, k)
    fb = eng.last_f32_fallback()
    eng.set_f32_datapath("3xtf32")
    g32 = eng.power(a, k)
    eng.set_f32_datapath("auto")
    return g16, fb, g32


@pytest.mark.parametrize("n,k", [(1024, 13), (1280, 9), (1500, 16), (2048, 7), (1024, 1000),
                                 (1600, 13), (2000, 9)])  # (1664 / 2048 padded to 1792 / 2048)
def test_k1ph_chain_vs_oracle_and_3xtf32(eng, n, k):
    a = oracle.scaled_input(n, np.float32, 42)
    g16, fb, g32 = _both(eng, a, k)
    assert not fb  # random inputs never lose range
    ref = oracle.exponentiate(a, k, oracle.max_threads())
    e16, e32 = oracle.compare(g16, ref)[2], oracle.compare(g32, ref)[2]
    assert np.isfinite(g16).all()
    assert e16 <= mx.fro_tol(n, k, "f32"), (n, k, e16)
    assert e16 <= 2.0 * e32 + 1e-7, (n, k, e16, e32)


def test_k1ph_not_used_off_pair_sizes(eng):
    """n = 1100 (n_pad 1152, inside K1C's one-launch range) stays on 3xTF32
    whatever the switch."""
    a = oracle.scaled_input(1100, np.float32, 5)
    eng.set_f32_datapath("auto")
    g16 = eng.power(a, 9)
    with pytest.raises(mx.UnsupportedError):  # no K1PH chain ran
        eng.last_f32_fallback()
    eng.set_f32_datapath("3xtf32")
    g32 = eng.power(a, 9)
    eng.set_f32_datapath("auto")
    assert g16.tobytes() == g32.tobytes()


def _cancelling(n, seed=5):
    rng = np.random.default_rng(seed)
    nil = np.zeros((n, n))
    nil[: n // 2, n // 2:] = rng.uniform(-1, 1, (n // 2, n // 2))
    return (nil + 1e-6 * rng.uniform(-1, 1, (n, n))).astype(np.float32)


@pytest.mark.parametrize("n", [1024, 1536, 1600])  # 1600: K1PH at 1792, recomputation on K1 at 1664
def test_k1ph_cancellation_recomputed_on_3xtf32(eng, n):
    """A = N + eps R, N^2 = 0: A^2 ~ eps, so the one-exponent planes would
    lose the eps^2 entries A^6 depends on.  The split of A^2 raises the flag
    and the gated 3xTF32 chain recomputes the power: the result is bitwise the
    3xTF32 datapath's."""
    a = _cancelling(n)
    for k in (3, 6):
        g16, fb, g32 = _both(eng, a, k)
        assert fb, (n, k)
        assert g16.tobytes() == g32.tobytes(), (n, k)
        exact = np.linalg.matrix_power(a.astype(np.float64), k)
        ref = oracle.exponentiate(a, k, oracle.max_threads())
        d = lambda x, y: float(np.linalg.norm(x.astype(np.float64) - y) / np.linalg.norm(y))  # noqa: E731
        assert d(g16, exact) <= max(mx.fro_tol_conditioned(n, k, "f32"), 64 * d(ref, exact))


def test_k1ph_nan_zero_and_exact_inputs(eng):
    n = 1024
    # NaN: non-finite product -> recomputed on 3xTF32 (the reference's NaN pattern)
    a = oracle.scaled_input(n, np.float32, 3)
    a[7, 9] = np.nan
    g16, fb, g32 = _both(eng, a, 3)
    assert fb and np.array_equal(np.isnan(g16), np.isnan(g32))
    # an inf in the base, one-step plan (no product is split): the base split
    # raises the flag, so the result carries the 3xTF32 chain's inf / NaN pattern
    b = oracle.scaled_input(n, np.float32, 4)
    b[3, 5] = np.inf
    g16, fb, g32 = _both(eng, b, 2)
    assert fb and g16.tobytes() == g32.tobytes()
    # zero matrix: zero product, exact zeros
    z = np.zeros((n, n), np.float32)
    g16, fb, _ = _both(eng, z, 13)
    assert not g16.any()
    # signed permutation: exact in scaled fp16 (one exponent, entries +-1)
    rng = np.random.default_rng(11)
    p = np.zeros((n, n), np.float32)
    p[np.arange(n), rng.permutation(n)] = rng.choice([-1.0, 1.0], n).astype(np.float32)
    want = np.linalg.matrix_power(p.astype(np.float64), 37).astype(np.float32)
    g16, fb, _ = _both(eng, p, 37)
    assert np.array_equal(g16, want)


def test_k1ph_scale_range(eng):
    """Powers that grow / shrink by many orders of magnitude: the per-matrix
    exponent follows them exactly (products of 1e15 and 1e-15 inputs)."""
    n = 1024
    base = oracle.scaled_input(n, np.float32, 8)
    for s, k in ((1e15, 2), (1e-15, 2), (1e3, 5), (1e-3, 5)):
        a = (base * np.float32(s)).astype(np.float32)
        g16, fb, g32 = _both(eng, a, k)
        ref = oracle.exponentiate(a, k, oracle.max_threads())
        if not np.isfinite(ref).all() or not ref.any():
            continue
        assert oracle.compare(g16, ref)[2] <= mx.fro_tol(n, k, "f32"), (s, k)


def test_datapath_switch_validation(eng):
    with pytest.raises(ValueError):
        eng.set_f32_datapath("fp8")
    eng.set_f32_datapath("3xtf32")
    eng.set_f32_datapath("auto")


@pytest.mark.parametrize("n,k", [(1024, 2), (1024, 3), (1100 + 700, 2), (8200, 2)])
def test_k1ph_short_chains_and_large_ragged(eng, n, k):
    """One- and two-step plans (the last GEMM writes the result straight from
    K1PH's epilogue; no split is tested for range) and ragged orders padded to
    256 (8200 -> 8448): vs the oracle."""
    a = oracle.scaled_input(n, np.float32, 7)
    eng.set_f32_datapath("auto")
    got = eng.power(a, k)
    assert not eng.last_f32_fallback()
    ref = oracle.exponentiate(a, k, oracle.max_threads())
    assert oracle.compare(got, ref)[2] <= mx.fro_tol(n, k, "f32")


def test_k1ph_graph_cache_across_datapath_switches(eng):
    """Cached chain graphs are dropped when the datapath changes: alternating
    switches reproduce each datapath's own result bitwise."""
    a = oracle.scaled_input(1024, np.float32, 9)
    eng.set_f32_datapath("auto")
    want16 = eng.power(a, 13)
    eng.set_f32_datapath("3xtf32")
    want32 = eng.power(a, 13)
    assert want16.tobytes() != want32.tobytes()
    for _ in range(2):
        eng.set_f32_datapath("auto")
        assert eng.power(a, 13).tobytes() == want16.tobytes()
        eng.set_f32_datapath("3xtf32")
        assert eng.power(a, 13).tobytes() == want32.tobytes()
    eng.set_f32_datapath("auto")


def test_k1ph_batched_chains(eng):
    """mxp_power_batched with n > 128 runs one chain per matrix (K1PH at these
    sizes): each matrix as its own single chain, bitwise."""
    stack = np.stack([oracle.scaled_input(1024, np.float32, 20 + i) for i in range(3)])
    out = eng.power_batched(stack, 9)
    for i in range(3):
        assert out[i].tobytes() == eng.power(stack[i], 9).tobytes()
