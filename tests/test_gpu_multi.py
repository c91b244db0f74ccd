"""mxp_power_multi: several devices from one process (batch shards; one
matrix row-sharded with the exchange fused into the CTA-pair epilogue, CUDA
events between steps).  The box has one GPU, so the "devices" are the same
B200 listed several times — every occurrence gets its own handle and stream,
so the sharding, the peer stores into other handles' buffers and the
cross-stream step ordering run exactly as across GPUs (only the NVLink hop is
missing).  Batch shards and row shards must be BITWISE the single-device
results (same kernels, same per-element order)."""

import math

import numpy as np
import pytest

import oracle
import paper_1204_3052_b200 as mx
from paper_1204_3052_b200 import engine as E

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    e = mx.Engine(0)
    # the row-sharded FP32 chains run 3xTF32 (an exponent per element); the
    # single-device reference runs the same datapath so results are bitwise
    e.set_f32_datapath("3xtf32")
    yield e
    E.release_multi()


def _batch(n, b, dt=np.float32, seed=42):
    return np.stack([oracle.scaled_input(n, dt, seed + i) for i in range(b)])


@pytest.mark.parametrize("devices,n,b,k", [
    ([0, 0], 128, 1000, 64),      # C3 shape, two shards (K3H)
    ([0, 0, 0], 64, 7, 1000),     # uneven shards, K3B route
    ([0, 0, 0, 0], 200, 5, 13),   # n > 128: per-matrix chains, one empty-ish shard
    ([0, 0], 96, 3, 0),           # k = 0 -> identities
])
def test_batch_shards_bitwise_single_device(eng, devices, n, b, k):
    a = _batch(n, b)
    got = mx.exponentiate_multi(a, k, devices)
    ref = eng.power_batched(a, k)
    assert got.tobytes() == ref.tobytes()
    st = E.power_multi.last_stats
    assert st.multiply_count == mx.multiply_count(k) * b
    assert st.h2d == min(len(devices), b) and st.d2h == min(len(devices), b)


def test_batch_shards_f64(eng):
    a = _batch(48, 6, np.float64)
    got = mx.exponentiate_multi(a, 9, [0, 0])
    assert got.tobytes() == eng.power_batched(a, 9).tobytes()


@pytest.fixture(scope="module")
def eng_auto():
    """The default datapath: K1PH at the CTA-pair sizes (what the row shards
    run there)."""
    return mx.Engine(0)


@pytest.mark.parametrize("devices,n,k", [
    ([0, 0], 1024, 13),        # n_p = 1024 = the single chain's K1PH order: bitwise
    ([0, 0, 0, 0], 2048, 16),  # four row blocks of 512
    ([0, 0, 0], 1500, 13),     # ragged: 1500 -> 3 x 512 rows (single chain: n_pad 1536)
    ([0, 0], 1600, 9),         # 1600 -> 2 x 1024 rows (single chain: 1792; padding adds exact zeros)
    ([0, 0, 0], 1024, 2),      # a one-step plan; 1024 -> 3 x 512 rows (1536, padding rows only on the last)
])
def test_row_shards_bitwise_single_device(eng_auto, devices, n, k):
    """K1PH row shards: each device's rows from the K1PH row-block GEMM, the
    maxima met in every device's state, every device's rows split at the
    global exact scale into every device's planes — bitwise the single-device
    K1PH chain."""
    a = oracle.scaled_input(n, np.float32, 42)
    got = mx.exponentiate_multi(a, k, devices)
    ref = eng_auto.power(a, k)
    assert not eng_auto.last_f32_fallback()
    assert got.tobytes() == ref.tobytes()
    st = E.power_multi.last_stats
    assert st.multiply_count == mx.multiply_count(k)
    assert st.h2d == len(devices) and st.d2h == 1
    err = oracle.compare(got, oracle.exponentiate(a, k, oracle.max_threads()))[2]
    assert err <= mx.fro_tol(n, k, "f32"), err


@pytest.mark.parametrize("devices,n", [([0, 0], 1024), ([0, 0, 0], 1536)])
def test_row_shards_cancellation_recomputed_on_3xtf32(eng, eng_auto, devices, n):
    """A product that loses dynamic range (A = N + 1e-6 R, N^2 = 0) makes the
    K1PH row shards recompute on the 3xTF32 row shards: bitwise the 3xTF32
    single-device chain, and the default single-device chain (which falls
    back the same way)."""
    rng = np.random.default_rng(5)
    nil = np.zeros((n, n))
    nil[: n // 2, n // 2:] = rng.uniform(-1, 1, (n // 2, n // 2))
    a = (nil + 1e-6 * rng.uniform(-1, 1, (n, n))).astype(np.float32)
    got = mx.exponentiate_multi(a, 6, devices)
    assert got.tobytes() == eng.power(a, 6).tobytes()   # eng: MXP_DATAPATH_3XTF32
    auto = eng_auto.power(a, 6)
    assert eng_auto.last_f32_fallback()
    assert got.tobytes() == auto.tobytes()


def test_row_shards_small_order_vs_oracle(eng):
    """n = 300 pads to the pair kernel's 1024 rows (the single chain runs K1C
    at n_pad 384, so parity is by tolerance, not bitwise)."""
    a = oracle.scaled_input(300, np.float32, 7)
    got = mx.exponentiate_multi(a, 100, [0, 0])
    err = oracle.compare(got, oracle.exponentiate(a, 100, oracle.max_threads()))[2]
    assert np.isfinite(got).all()
    assert err <= mx.fro_tol(300, 100, "f32"), err


@pytest.mark.parametrize("devices,n,k", [([0, 0], 256, 9), ([0, 0, 0], 1000, 13),
                                         ([0, 0, 0, 0], 600, 257)])
def test_row_shards_f64_bitwise_single_device(eng, devices, n, k):
    """FP64: DMMA row-block GEMMs + peer copies of each device's rows."""
    a = oracle.scaled_input(n, np.float64, 42)
    got = mx.exponentiate_multi(a, k, devices)
    assert got.tobytes() == eng.power(a, k).tobytes()
    st = E.power_multi.last_stats
    assert st.multiply_count == mx.multiply_count(k) and st.h2d == len(devices) and st.d2h == 1


def test_replica_cases_equal_mxp_power(eng):
    """n <= 128 FP32, small FP64 and k <= 1 run on devices[0] alone."""
    for n, dt, k in ((64, np.float32, 16), (200, np.float64, 9), (300, np.float32, 1),
                     (300, np.float32, 0)):
        a = oracle.scaled_input(n, dt, 3)
        got = mx.exponentiate_multi(a, k, [0, 0])
        assert got.tobytes() == eng.power(a, k).tobytes(), (n, dt, k)


def test_exact_inputs_row_sharded(eng):
    """A signed permutation (exact in 3xTF32): P^k through the row-sharded
    chain equals the exact integer power."""
    n = 1024
    rng = np.random.default_rng(5)
    perm = rng.permutation(n)
    p = np.zeros((n, n), np.float32)
    p[np.arange(n), perm] = rng.choice([-1.0, 1.0], n).astype(np.float32)
    k = 37
    ref = np.eye(n, dtype=np.float32)
    for _ in range(k):
        ref = (ref.astype(np.float64) @ p.astype(np.float64)).astype(np.float32)
    got = mx.exponentiate_multi(p, k, [0, 0, 0, 0])
    assert np.array_equal(got, ref)


def test_more_devices_than_matrices_and_bad_ordinals(eng):
    """batch < ngpus uses one device per matrix; an ordinal the machine does
    not have is a validation error before any work (no silent fallback)."""
    a = _batch(64, 2)
    got = mx.exponentiate_multi(a, 16, [0, 0, 0])
    assert got.tobytes() == eng.power_batched(a, 16).tobytes()
    assert E.power_multi.last_stats.h2d == 2
    with pytest.raises(mx.ValidationError):
        mx.exponentiate_multi(a, 16, [0, E.device_count()])
    with pytest.raises(mx.ValidationError):
        mx.exponentiate_multi(oracle.scaled_input(512, np.float32, 1), 4, [0] * 9)
