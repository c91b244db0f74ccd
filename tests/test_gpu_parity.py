"""GPU parity: the sm_100a engine (through the C ABI) against the CPU oracle
and the reference's golden fixtures.  Run on a B200 (`pytest -m gpu`).

Tolerances (written here, derived in SURVEY §8(d) / DESIGN.md):
* one multiply: max_rel <= n * u * 64  (reference device_tol, tolerances.py:316-319)
* A^k chains:   frobenius_rel <= 16 * m(k) * sqrt(n) * u  (m(k) = multiply count)
* exact inputs (Fibonacci, permutations): bitwise.
"""

import hashlib
import math

import numpy as np
import pytest

import oracle
import paper_1204_3052_b200 as mx
from paper_1204_3052_b200 import _lib
from paper_1204_3052_b200.engine import Engine

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24
U64 = 2.0 ** -53


@pytest.fixture(scope="module")
def eng():
    e = Engine(0)
    yield e
    e.close()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fro(res, ref):
    return oracle.compare(res, ref)[2]


# ------------------------------------------------------------------ generation
def test_device_random_matrix_bitexact(golden):
    arrays, meta = golden
    for key in arrays.files:
        if not key.startswith("rm_"):
            continue
        _, n, dt, seed, lo, hi = key.split("_")
        dtype = mx.DType.F32 if dt == "f32" else mx.DType.F64
        got = mx.random_matrix(int(n), dtype, int(seed), float(lo), float(hi)).array
        assert got.tobytes() == arrays[key].tobytes(), key
    for key, digest in meta["random_matrix_sha256"].items():
        n, dt, seed = key.split("_")
        dtype = mx.DType.F32 if dt == "f32" else mx.DType.F64
        assert sha(mx.random_matrix(int(n), dtype, int(seed)).array) == digest, key


def test_splitmix64_exported_and_bitexact(golden):
    """splitmix64 is public API in the reference (linalg.py:117-124, __all__); its
    frozen KATs (test_linalg.py:28-45) and the golden streams, through ours."""
    arrays, _ = golden
    kats = {0: (0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC),
            42: (0xBDD732262FEB6E95, 0x28EFE333B266F103, 0x47526757130F9F52, 0x581CE1FF0E4AE394),
            2024: (0x9F6D8FECF88EECD5, 0x18E430BB1511F2D2, 0x4C6F7CBF58DBA57F, 0x1DBE69E0AE9BB859)}
    for seed, want in kats.items():
        got = mx.splitmix64(seed, 4)
        assert got.dtype == np.uint64 and tuple(int(v) for v in got) == want
    for seed in (0, 42, 2024, 7, 2**64 - 1):
        assert np.array_equal(mx.splitmix64(seed, 16), arrays[f"sm64_{seed}"])
    big = mx.splitmix64(123, 1 << 20)
    assert np.array_equal(big, oracle.splitmix64(123, 1 << 20))
    assert mx.splitmix64(5, 0).shape == (0,)


def test_device_scaled_recipe_bitexact(golden):
    _, meta = golden
    for key, digest in meta["scaled_sha256"].items():
        n, dt, seed = key.split("_")
        dtype = mx.DType.F32 if dt == "f32" else mx.DType.F64
        assert sha(mx.scaled_input(int(n), dtype, int(seed)).array) == digest, key
    stack = mx.scaled_batch(128, 3, mx.DType.F32, 42)
    for i in range(3):
        assert stack[i].tobytes() == oracle.scaled_input(128, np.float32, 42 + i).tobytes()


# ------------------------------------------------------------------ one multiply
@pytest.mark.parametrize("n", [1, 7, 64, 128, 200, 256, 384, 512, 1024])
def test_multiply_f32_device_tol(eng, n):
    a = oracle.random_matrix(n, np.float32, 1000 + n)
    b = oracle.random_matrix(n, np.float32, 2000 + n)
    got = eng.multiply(a, b)
    ref = oracle.matmul(a, b)
    _, max_rel, _ = oracle.compare(got, ref)
    assert max_rel <= n * U32 * 64, (n, max_rel)
    st = eng.last_stats
    assert st.multiply_count == 1 and st.h2d == 2 and st.d2h == 1


@pytest.mark.parametrize("n", [1, 5, 64, 200, 256])
def test_multiply_f64_device_tol(eng, n):
    a = oracle.random_matrix(n, np.float64, 1000 + n)
    b = oracle.random_matrix(n, np.float64, 2000 + n)
    got = eng.multiply(a, b)
    ref = oracle.matmul(a, b)
    assert oracle.compare(got, ref)[1] <= n * U64 * 64


def test_multiply_identity_within_rounding(eng):
    """host.test.ts:92-100: A*I within n*2^-24*max|A|."""
    n = 32
    a = oracle.random_matrix(n, np.float32, 77)
    got = eng.multiply(a, np.eye(n, dtype=np.float32))
    assert np.abs(got - a).max() <= n * U32 * np.abs(a).max()


# ------------------------------------------------------------------ chains vs golden
@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("n", [2, 4, 8, 16, 64])
def test_exponentiate_vs_reference_golden(golden, dt, n):
    arrays, _ = golden
    dtype = mx.DType.F32 if dt == "f32" else mx.DType.F64
    u = dtype.roundoff
    a = mx.Matrix(arrays[f"in_{n}_{dt}"])
    for k in (0, 1, 2, 3, 7, 13, 16, 64):
        got = mx.exponentiate(a, k, mx.b200_backend())
        ref = arrays[f"exp_{n}_{dt}_{k}"]
        if k <= 1:
            assert got.array.tobytes() == ref.tobytes(), (n, dt, k)
            continue
        tol = 16 * mx.multiply_count(k) * math.sqrt(n) * u
        assert fro(got.array, ref) <= tol, (n, dt, k, fro(got.array, ref), tol)


def test_power_one_returns_same_object_and_zero_multiplies(eng):
    a = mx.Matrix(oracle.random_matrix(32, np.float32, 6))
    assert mx.exponentiate(a, 1, mx.b200_backend()) is a
    out = eng.power(a.array, 1)
    assert out.tobytes() == a.array.tobytes()
    assert eng.last_stats.multiply_count == 0 and eng.last_stats.launches == 0
    assert eng.last_stats.h2d == 1 and eng.last_stats.d2h == 1


def test_power_zero_is_identity(eng):
    for dt in (np.float32, np.float64):
        out = eng.power(oracle.random_matrix(7, dt, 1), 0)
        assert np.array_equal(out, np.eye(7, dtype=dt))


def test_fibonacci_exact_through_device_chain(golden):
    """host.test.ts:157-171 (4x4 block-embedded, f32) and the f64 KATs."""
    arrays, _ = golden
    q = np.zeros((4, 4), dtype=np.float32)
    q[:2, :2] = [[1, 1], [1, 0]]
    q[2, 2] = q[3, 3] = 1
    eng = mx.Engine(0)
    got = eng.power(q, 10)
    assert got[0, 0] == 89 and got[0, 1] == 55 and got[1, 0] == 55 and got[1, 1] == 34
    assert eng.last_stats.multiply_count == 4
    q64 = np.array([[1.0, 1.0], [1.0, 0.0]])
    for k in (10, 40, 78):
        assert np.array_equal(eng.power(q64, k), arrays[f"fib_f64_{k}"]), k
    # F_40 < 2^24: exact in f32 too (3xTF32 splits small integers exactly)
    assert np.array_equal(eng.power(q64.astype(np.float32), 30), oracle.exponentiate(
        q64.astype(np.float32), 30))


def test_well_conditioned_chain_vs_f64_repeated(golden):
    """host.test.ts:173-184: n=64, k=64, maxRel <= k*n*2^-24*64, 6 multiplies."""
    arrays, _ = golden
    eng = mx.Engine(0)
    got = eng.power(arrays["wc_in_64_f32"], 64)
    rel = oracle.compare(got, arrays["wc_rep64_64_f64"])[1]
    assert np.isfinite(rel) and rel <= 64 * 64 * U32 * 64
    assert eng.last_stats.multiply_count == 6


def test_transfer_and_count_laws(eng):
    a = oracle.random_matrix(16, np.float32, 3) * np.float32(0.2)
    for k in (1, 2, 13, 1024):
        eng.power(a, k)
        st = eng.last_stats
        assert st.h2d == 1 and st.d2h == 1
        assert st.multiply_count == mx.multiply_count(k)


def test_validation_before_device_work(eng):
    with pytest.raises(ValueError):
        eng.power(np.zeros((4, 4), np.float32), -1)
    with pytest.raises(ValueError):
        eng.multiply(np.zeros((4, 4), np.float32), np.zeros((5, 5), np.float32))
    with pytest.raises(ValueError):
        eng.multiply(np.zeros((4, 4), np.float32), np.zeros((4, 4), np.float64))
    with pytest.raises(mx.ShapeError):
        eng.power(np.zeros((4, 4), np.int64), 3)


def test_backend_interop_and_counting():
    be = mx.CountingBackend(mx.b200_backend())
    a = mx.Matrix(oracle.scaled_input(64, np.float32, 42))
    out = mx.exponentiate(a, 13, be)
    assert be.calls == 5
    ref = oracle.exponentiate(a.array, 13)
    assert fro(out.array, ref) <= 16 * 5 * 8 * U32


# ------------------------------------------------------------------ configs
def test_config1_64_a16(golden):
    arrays, _ = golden
    a = oracle.scaled_input(64, np.float32, 42)
    got = mx.Engine(0).power(a, 16)
    assert fro(got, arrays["exp_64_f32_16"]) <= mx.fro_tol(64, 16, "f32")
    # the reference's own unscaled default input (finite at k=16)
    got = mx.Engine(0).power(arrays["unscaled_in_64_f32"], 16)
    assert fro(got, arrays["unscaled_exp_64_f32_16"]) <= mx.fro_tol(64, 16, "f32")


def test_config2_512_a1000():
    a = oracle.scaled_input(512, np.float32, 42)
    ref = oracle.exponentiate(a, 1000)
    got = mx.Engine(0).power(a, 1000)
    assert np.isfinite(got).all()
    assert fro(got, ref) <= mx.fro_tol(512, 1000, "f32"), fro(got, ref)


def test_config3_batched_samples(golden):
    """128x128 A^64, seeds 42+i, generated on device, chained in the persistent kernel
    through the host API (chunked pipeline: launches of <= 1024 matrices, about 3-4
    per chain).  The bench's exact launch (all 65536 matrices in one launch, ~221
    per chain) is checked matrix by matrix in tests/test_gpu_configs.py."""
    arrays, meta = golden
    batch = 4352
    stack = mx.scaled_batch(128, batch, mx.DType.F32, 42)
    out = mx.exponentiate_batched(stack, 64)
    tol = mx.fro_tol(128, 64, "f32")
    assert fro(out[0], arrays["c3_out_0"]) <= tol
    for i in (1, 255, 4097):
        ref = oracle.exponentiate(oracle.scaled_input(128, np.float32, 42 + i), 64)
        assert sha(ref) == meta["c3_exp_sha256"][str(i)]
        assert fro(out[i], ref) <= tol, i
    # batched result is bitwise the single-matrix result (same kernel, same order)
    single = mx.Engine(0).power(stack[255], 64)
    assert single.tobytes() == out[255].tobytes()


def test_batched_small_n_with_multiplies():
    """n < 128 and plans with MULTIPLY_BASE steps in the persistent kernel."""
    for n, k in ((5, 1000), (33, 13), (100, 13), (128, 257), (127, 7)):
        stack = mx.scaled_batch(n, 300, mx.DType.F32, 7)
        if k > 100:  # keep A^k finite: row-stochastic inputs (spectral radius 1)
            st = np.abs(stack).astype(np.float64)
            stack = (st / st.sum(axis=2, keepdims=True)).astype(np.float32)
        out = mx.exponentiate_batched(stack, k)
        for i in (0, 151, 299):
            ref = oracle.exponentiate(stack[i], k)
            assert fro(out[i], ref) <= mx.fro_tol_conditioned(n, k, "f32"), (n, k, i)


def test_batched_into_caller_out():
    """exponentiate_batched(..., out=) writes into the caller's array, bitwise
    the fresh-result call; a wrong out is rejected before any device work."""
    stack = mx.scaled_batch(128, 200, mx.DType.F32, 11)
    ref = mx.exponentiate_batched(stack, 64)
    out = np.full_like(stack, np.nan)
    got = mx.exponentiate_batched(stack, 64, out=out)
    assert got is out and out.tobytes() == ref.tobytes()
    with pytest.raises(mx.ShapeError):
        mx.exponentiate_batched(stack, 64, out=np.empty((200, 128, 127), np.float32))
    with pytest.raises(mx.ShapeError):
        mx.exponentiate_batched(stack, 64, out=np.empty_like(stack, dtype=np.float64))


def test_large_chain_with_multiplies_f32():
    for n, k in ((200, 13), (256, 257), (384, 100)):
        a = oracle.scaled_input(n, np.float32, 42)
        got = mx.Engine(0).power(a, k)
        ref = oracle.exponentiate(a, k)
        assert fro(got, ref) <= mx.fro_tol_conditioned(n, k, "f32"), (n, k, fro(got, ref))


def test_f64_chain_256_a257(golden):
    _, meta = golden
    a = oracle.scaled_input(256, np.float64, 42)
    ref = oracle.exponentiate(a, 257)
    assert sha(ref) == meta["exp_256_f64_257_sha256"]
    got = mx.Engine(0).power(a, 257)
    assert fro(got, ref) <= mx.fro_tol(256, 257, "f64"), fro(got, ref)


def test_stochastic_matrix_power_1000(golden):
    arrays, _ = golden
    got = mx.Engine(0).power(arrays["stoch_in_5_f32"], 1000)
    assert fro(got, arrays["stoch_exp_5_f32_1000"]) <= mx.fro_tol_conditioned(5, 1000, "f32")


# ------------------------------------------------------------------ full-size properties
def test_permutation_power_exact_8192():
    """Size-independent property at the C5 size: a permutation matrix of
    order 12 (disjoint 3- and 4-cycles) raised to 1024 = 12*85 + 4 equals
    P^4 exactly (0/1 entries are exact in 3xTF32)."""
    n = 8192
    perm = np.arange(n)
    for base in range(0, n - 7, 7):
        perm[base:base + 3] = np.roll(perm[base:base + 3], 1)
        perm[base + 3:base + 7] = np.roll(perm[base + 3:base + 7], 1)
    p = np.zeros((n, n), dtype=np.float32)
    p[np.arange(n), perm] = 1.0
    eng = mx.Engine(0)
    got = eng.power(p, 1024)
    p4 = np.arange(n)
    for _ in range(4):
        p4 = perm[p4]
    ref = np.zeros((n, n), dtype=np.float32)
    ref[np.arange(n), p4] = 1.0
    assert np.array_equal(got, ref)
    assert eng.last_stats.multiply_count == 10


def test_row_stochastic_8192_a1024():
    """Row sums of a row-stochastic matrix stay 1 under any power."""
    n = 8192
    eng = mx.Engine(0)
    a = np.abs(mx.scaled_batch(n, 1, mx.DType.F32, 42)[0]).astype(np.float64)
    a = (a / a.sum(axis=1, keepdims=True)).astype(np.float32)
    got = eng.power(a, 1024)
    sums = got.astype(np.float64).sum(axis=1)
    assert np.abs(sums - 1.0).max() <= 16 * 10 * math.sqrt(n) * U32


# ------------------------------------------------------------------ exact modular mode
@pytest.mark.parametrize("n,k,p", [(2, 60, 10), (5, 6, 97), (64, 13, 2**31 - 1), (130, 257, 65521),
                                   (200, 1000, 1000003), (1, 5, 7), (257, 2, 2**31 - 1)])
def test_modular_bitexact_vs_oracle(eng, n, k, p):
    rng = np.random.default_rng(n * 1000 + k)
    a = rng.integers(0, 2**32 - 1, size=(n, n), dtype=np.uint64).astype(np.uint32)
    got = eng.power_mod(a, k, p)
    ref = oracle.exponentiate_mod(a, k, p)
    assert np.array_equal(got, ref), (n, k, p)
    assert eng.last_stats.multiply_count == mx.multiply_count(k)


@pytest.mark.parametrize("n,k,p", [(128, 13, 2**31 - 1), (384, 33, 2147483629), (1000, 9, 65537),
                                   (1024, 257, 2**31 - 1), (129, 64, 3), (256, 5, 2)])
def test_modular_int8_datapath_bitexact(eng, n, k, p):
    """The INT8 tensor-core path (K5I: byte limbs, s32 diagonal accumulators,
    Barrett folding) against the exact oracle: ragged n, moduli near 2^31
    (every limb byte populated), tiny moduli, and long plans."""
    rng = np.random.default_rng(n + k)
    a = rng.integers(0, 2**32 - 1, size=(n, n), dtype=np.uint64).astype(np.uint32)
    got = eng.power_mod(a, k, p)
    ref = oracle.exponentiate_mod(a, k, p, oracle.max_threads())
    assert np.array_equal(got, ref), (n, k, p, int((got != ref).sum()))


def test_modular_worst_case_accumulators_8192(eng):
    """n = 8192 (the largest order on the INT8 path) with every residue = p - 1
    for p = 2^31 - 1: every limb byte is 0xFF except the top one (0x7F), so the
    diagonal accumulators reach 4 n 255^2 - ... close to 2^31 without wrapping.
    (p-1) J squared is n (p-1)^2 J = n J (mod p): checked against exact ints."""
    n, p = 8192, 2**31 - 1
    a = np.full((n, n), p - 1, dtype=np.uint32)
    got = eng.power_mod(a, 2, p)
    assert np.all(got == n % p)
    got = eng.power_mod(a, 3, p)  # n^2 (p-1)^3 J = -n^2 J
    assert np.all(got == (-(n * n)) % p)


def test_modular_dmma_path_beyond_int8_range(eng):
    """n > 8192 runs the FP64 DMMA Karatsuba path: a permutation of order 12
    at n = 8200 (and its powers) exactly."""
    n = 8200
    perm = np.arange(n)
    for base in range(0, n - 7, 7):
        perm[base:base + 3] = np.roll(perm[base:base + 3], 1)
        perm[base + 3:base + 7] = np.roll(perm[base + 3:base + 7], 1)
    pm = np.zeros((n, n), dtype=np.uint32)
    pm[np.arange(n), perm] = 1
    assert np.array_equal(eng.power_mod(pm, 12, 1000003), np.eye(n, dtype=np.uint32))
    p5 = np.arange(n)
    for _ in range(5):
        p5 = perm[p5]
    want = np.zeros((n, n), dtype=np.uint32)
    want[np.arange(n), p5] = 7
    assert np.array_equal(eng.power_mod(pm * np.uint32(7), 5, 2**31 - 1) % np.uint32(2**31 - 1),
                          (want.astype(np.uint64) * 7**4 % (2**31 - 1)).astype(np.uint32))


def test_modular_kats(eng):
    q = np.array([[1, 1], [1, 0]], dtype=np.uint32)
    assert np.array_equal(eng.power_mod(q, 60, 10), np.eye(2))      # Pisano period pi(10) = 60
    assert np.array_equal(eng.power_mod(q, 16, 7), np.eye(2))       # pi(7) = 16
    fib = [0, 1]
    for _ in range(200):
        fib.append(fib[-1] + fib[-2])
    p = 2**31 - 1
    got = eng.power_mod(q, 150, p)
    assert int(got[0, 1]) == fib[150] % p and int(got[0, 0]) == fib[151] % p
    n = 4096  # permutation of order 12 at a large size: P^12 == I exactly
    perm = np.arange(n)
    for base in range(0, n - 7, 7):
        perm[base:base + 3] = np.roll(perm[base:base + 3], 1)
        perm[base + 3:base + 7] = np.roll(perm[base + 3:base + 7], 1)
    pm = np.zeros((n, n), dtype=np.uint32)
    pm[np.arange(n), perm] = 1
    assert np.array_equal(eng.power_mod(pm, 12, 1000003), np.eye(n, dtype=np.uint32))
    assert np.array_equal(eng.power_mod(pm, 0, 5), np.eye(n, dtype=np.uint32))
    with pytest.raises(ValueError):
        eng.power_mod(q, 3, 1)


# ------------------------------------------------------------------ multi-GPU building blocks
@pytest.mark.parametrize("n,rows", [(256, 128), (300, 77), (8192, 1024)])
def test_gemm_rows_bitwise_equals_full_multiply(n, rows):
    """A row block of one multiply is bitwise the same rows of the full product
    (the property that makes row-sharded chains equal to single-GPU ones)."""
    import torch

    eng = mx.Engine(0)
    a = torch.from_numpy(oracle.random_matrix(n, np.float32, 3)).cuda()
    b = torch.from_numpy(oracle.random_matrix(n, np.float32, 4)).cuda()
    full = torch.empty_like(a)
    part = torch.empty((rows, n), dtype=a.dtype, device=a.device)
    r0 = n - rows
    eng.gemm_device(a.data_ptr(), b.data_ptr(), full.data_ptr(), n)
    eng.gemm_rows_device(a[r0:].contiguous().data_ptr(), b.data_ptr(), part.data_ptr(), n, rows)
    eng.synchronize()
    assert torch.equal(part, full[r0:])


@pytest.mark.parametrize("mode_dt", ["f32", "f64"])
def test_prepared_rhs_chunks_bitwise_and_invalidation(mode_dt):
    """mxp_gemm_prepare_rhs once + several mxp_gemm_rows_prepared row chunks ==
    the full multiply's rows, bitwise; any other workspace use invalidates the
    prepared right-hand side (validation error, not a silent stale result)."""
    import torch

    dt = np.float32 if mode_dt == "f32" else np.float64
    mode = _lib.MXP_F32 if mode_dt == "f32" else _lib.MXP_F64
    n, c = 1024, 256
    eng = mx.Engine(0)
    a = torch.from_numpy(oracle.random_matrix(n, dt, 5)).cuda()
    b = torch.from_numpy(oracle.random_matrix(n, dt, 6)).cuda()
    full = torch.empty_like(a)
    eng.gemm_device(a.data_ptr(), b.data_ptr(), full.data_ptr(), n, mode)
    eng.gemm_prepare_rhs_device(b.data_ptr(), n, mode)
    parts = [torch.empty((c, n), dtype=a.dtype, device=a.device) for _ in range(n // c)]
    for j, part in enumerate(parts):
        eng.gemm_rows_prepared_device(a[j * c:(j + 1) * c].data_ptr(), part.data_ptr(), n, c, mode)
    eng.synchronize()
    assert torch.equal(torch.cat(parts), full)
    eng.gemm_device(a.data_ptr(), b.data_ptr(), full.data_ptr(), n, mode)  # reuses the workspace
    with pytest.raises(ValueError):
        eng.gemm_rows_prepared_device(a.data_ptr(), parts[0].data_ptr(), n, c, mode)


def test_row_sharded_chain_single_rank_nccl():
    import os

    import torch
    import torch.distributed as dist

    from paper_1204_3052_b200 import distributed as D

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        # the row blocks run K1 (3xTF32, split-K 4 at n = 512): bitwise the plan
        # executed one public multiply (mxp_gemm, same K1 arithmetic) at a time
        a = torch.from_numpy(oracle.scaled_input(512, np.float32, 42)).cuda()
        got = D.exponentiate_row_sharded(a, 1000)
        torch.cuda.synchronize()
        eng = mx.Engine(0)
        acc, tmp = a.clone(), torch.empty_like(a)
        for step in mx.plan_exponentiation(1000).steps:
            eng.gemm_device(acc.data_ptr(), (acc if step is mx.Step.SQUARE else a).data_ptr(),
                            tmp.data_ptr(), 512)
            acc, tmp = tmp, acc
        eng.synchronize()
        assert torch.equal(got, acc)  # bitwise: same kernels, same order
        batch = torch.from_numpy(mx.scaled_batch(64, 10, mx.DType.F32, 1)).cuda()
        out = D.exponentiate_batched_sharded(batch, 64)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), mx.exponentiate_batched(batch.cpu().numpy(), 64))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ harness / CLI / oracle on device
def test_device_repeated_oracle_and_cli(capsys):
    from paper_1204_3052_b200 import cli, harness

    eng = mx.Engine(0)
    a = oracle.random_matrix(16, np.float64, 42)
    rep = eng.repeated_power(a, 13)
    ref = oracle.exponentiate(a, 13)
    assert oracle.compare(rep, ref)[1] <= oracle.oracle_tol(13, 16, np.float64)
    assert cli.main(["verify", "--size", "64", "--power", "13", "--dtype", "f32"]) == 0
    out = capsys.readouterr().out
    assert "verdict=PASS" in out and "backend=b200" in out
    assert cli.main(["verify", "--size", "512", "--power", "1000", "--dtype", "f32",
                     "--scaled"]) == 0
    recs = harness.run_benchmark(harness.BenchConfig(sizes=[64], powers=[16, 13], repetitions=2))
    assert {(r.strategy.value, r.multiply_count) for r in recs} == {
        ("repeated", 15), ("squared", 4), ("repeated", 12), ("squared", 5)}
    assert all(r.max_rel_err is not None and r.max_rel_err < 1e-3 for r in recs)


# ------------------------------------------------------------------ small-n kernel (K3H) edge cases
# K3H keeps the running power as 2^e * P' with P' in fp16 pieces; these pin the
# per-step power-of-two rescaling, the two-chain schedule and the TMA IO path.
@pytest.mark.parametrize("mag", [1e-15, 1e-6, 1.0, 1e6, 1e15])
def test_small_n_scaling_extreme_magnitudes(eng, mag):
    """Results scale exactly with the input's magnitude (power-of-two scales
    are exact), so huge and tiny inputs meet the same tolerance."""
    n, k = 64, 2
    a = (oracle.scaled_input(n, np.float64, 11) * mag).astype(np.float32)
    got = eng.power(a, k)
    ref = oracle.exponentiate(a, k)
    assert np.isfinite(got).all()
    assert fro(got, ref) <= mx.fro_tol(n, k, "f32"), (mag, fro(got, ref))


@pytest.mark.parametrize("growth", [0.5, 2.0])
def test_small_n_growing_and_shrinking_powers(eng, growth):
    """A^64 with spectral radius ~0.5 (result ~1e-19) or ~2 (~1e19): every
    step rescales, nothing under- or overflows in the fp16 planes."""
    n, k = 128, 64
    a = (oracle.scaled_input(n, np.float64, 12) * growth).astype(np.float32)
    got = eng.power(a, k)
    ref = oracle.exponentiate(a, k)
    assert np.isfinite(ref).all() and np.isfinite(got).all()
    assert fro(got, ref) <= mx.fro_tol(n, k, "f32"), fro(got, ref)


def test_small_n_zero_and_nan(eng):
    z = np.zeros((64, 64), dtype=np.float32)
    assert not eng.power(z, 13).any()
    a = oracle.scaled_input(32, np.float32, 13)
    a[3, 5] = np.nan
    got = eng.power(a, 4)
    ref = oracle.exponentiate(a, 4)
    assert np.array_equal(np.isnan(got), np.isnan(ref))


def test_batched_mixed_magnitudes_and_schedule_edges():
    """Per-matrix scales are independent; batch sizes around the CTA / chain
    boundaries (1, 149, 297) and a skewed large batch with MULTIPLY_BASE steps."""
    n = 128
    for batch, k in ((1, 64), (149, 7), (297, 2), (1200, 13), (1200, 3)):
        stack = mx.scaled_batch(n, batch, mx.DType.F32, 21).astype(np.float64)
        e_max = max(1, 60 // k)  # |A_i^k| stays within 2^+-60 of the unscaled power
        scale = 2.0 ** ((np.arange(batch) % (2 * e_max + 1)) - e_max)
        stack = (stack * scale[:, None, None]).astype(np.float32)
        out = mx.exponentiate_batched(stack, k)
        for i in sorted({0, batch // 2, batch - 1, min(148, batch - 1)}):
            ref = oracle.exponentiate(stack[i], k)
            assert np.isfinite(out[i]).all()
            assert fro(out[i], ref) <= mx.fro_tol(n, k, "f32"), (batch, k, i, fro(out[i], ref))
        # deterministic: a second launch is bitwise identical
        assert np.array_equal(mx.exponentiate_batched(stack, k), out)


# ------------------------------------------------- one-launch chain (K1C)
@pytest.mark.parametrize("n,k", [(384, 33), (600, 7), (896, 9), (1300, 13)])
def test_one_launch_chain_bitwise_equals_single_multiplies(eng, n, k):
    """K1C (the 3xTF32 one-launch chain: n_pad 384, 640, 896, 1408 here) must
    be bitwise the same as the plan executed one public multiply at a time
    (mxp_gemm: split, one K1 GEMM with the same split-K and reduction order,
    fp32 out), following expo.py:131-138 with the accumulator on the left."""
    import torch

    a = torch.from_numpy(oracle.scaled_input(n, np.float32, 42)).cuda()
    chain = torch.empty_like(a)
    eng.power_device(a.data_ptr(), chain.data_ptr(), n, k)
    assert eng.last_stats.launches == 2  # split + one chain launch
    acc, tmp = a.clone(), torch.empty_like(a)
    for step in mx.plan_exponentiation(k).steps:
        rhs = acc if step is mx.Step.SQUARE else a
        eng.gemm_device(acc.data_ptr(), rhs.data_ptr(), tmp.data_ptr(), n)
        acc, tmp = tmp, acc
    eng.synchronize()
    assert torch.equal(chain, acc), (n, k)


@pytest.mark.parametrize("n", [129, 200, 255, 257, 384, 511, 640, 768, 896, 1100, 1300])
@pytest.mark.parametrize("k", [2, 3, 13])
def test_one_launch_chain_sizes_vs_exact(eng, n, k):
    """K1C over its whole size range (ragged n, split-K S = 1/2/4, plans with
    and without MULTIPLY_BASE steps) against the exact product in f64, within
    the chain tolerance."""
    a = oracle.scaled_input(n, np.float32, 7)
    got = eng.power(a, k)
    exact = np.linalg.matrix_power(a.astype(np.float64), k)
    assert np.isfinite(got).all()
    assert fro(got, exact) <= mx.fro_tol(n, k, "f32"), (n, k, fro(got, exact))
    assert eng.last_stats.launches == 2
    assert eng.last_stats.multiply_count == mx.plan_exponentiation(k).multiply_count


def test_result_independent_of_handle_history():
    """A handle that served a larger order first must run a small chain at the
    small order: same bits and same launch count as a fresh handle (the
    workspace is reused, never the larger padding)."""
    a = oracle.scaled_input(200, np.float32, 11)
    fresh = Engine(0)
    want = fresh.power(a, 13)
    want_launches = fresh.last_stats.launches
    fresh.close()
    used = Engine(0)
    used.multiply(oracle.scaled_input(1024, np.float32, 1), oracle.scaled_input(1024, np.float32, 2))
    got = used.power(a, 13)
    assert used.last_stats.launches == want_launches
    used.close()
    assert sha(got) == sha(want)


@pytest.mark.parametrize("batch,k", [(1200, 2), (1200, 4), (900, 5), (600, 64), (445, 3), (2000, 16)])
def test_batched_every_matrix_vs_oracle(batch, k):
    """Every matrix of the batch (not a sample) against the oracle: the K3H
    region rotation, the IO warp's next-boundary prediction and the skewed
    schedules must put every result in its place (plans of length 1-6, with
    and without MULTIPLY_BASE steps, batches around 3G and 4G)."""
    n = 128
    stack = mx.scaled_batch(n, batch, mx.DType.F32, 5)
    out = mx.exponentiate_batched(stack, k)
    ref = oracle.exponentiate_batched(stack, k, oracle.max_threads())
    tol = mx.fro_tol(n, k, "f32")
    diff = np.linalg.norm((out.astype(np.float64) - ref).reshape(batch, -1), axis=1)
    rel = diff / np.linalg.norm(ref.astype(np.float64).reshape(batch, -1), axis=1)
    assert np.isfinite(out).all()
    assert rel.max() <= tol, (batch, k, int(rel.argmax()), float(rel.max()), tol)


def test_batched_unaligned_device_pointers_take_the_scalar_path(eng):
    """n = 128 with 4-byte-misaligned device buffers: no TMA (the epilogue
    reads inputs and writes results itself); results bitwise equal to the
    aligned (TMA) run."""
    import torch

    n, batch, k = 128, 600, 13
    stack = mx.scaled_batch(n, batch, mx.DType.F32, 9)
    want = mx.exponentiate_batched(stack, k)
    src = torch.empty(batch * n * n + 1, dtype=torch.float32, device="cuda")
    dst = torch.empty(batch * n * n + 1, dtype=torch.float32, device="cuda")
    src[1:].copy_(torch.from_numpy(stack.reshape(-1)))
    eng.power_batched_device(src[1:].data_ptr(), dst[1:].data_ptr(), n, batch, k)
    eng.synchronize()
    got = dst[1:].cpu().numpy().reshape(batch, n, n)
    assert np.array_equal(got, want)


# ------------------------------------------------------------------ API hygiene
def test_cached_chain_replay_invalidates_prepared_rhs():
    """A chain replayed from the graph cache overwrites the workspace a prepared
    right-hand side lives in, so rows_prepared must refuse afterwards (cache
    miss and cache hit alike)."""
    import torch

    eng = mx.Engine(0)
    n = 512
    a = torch.from_numpy(oracle.scaled_input(n, np.float32, 3)).cuda()
    out = torch.empty_like(a)
    part = torch.empty((128, n), dtype=a.dtype, device=a.device)
    for _ in range(2):  # the second power_device replays the cached graph
        eng.gemm_prepare_rhs_device(a.data_ptr(), n)
        eng.power_device(a.data_ptr(), out.data_ptr(), n, 13)
        with pytest.raises(ValueError):
            eng.gemm_rows_prepared_device(a.data_ptr(), part.data_ptr(), n, 128)
    eng.synchronize()


def test_graph_cache_is_bounded_and_results_stay_right():
    """Fresh buffers on every call (as with torch tensors) capture a new graph
    each time; the cache evicts instead of growing, and replays stay correct."""
    import torch

    eng = mx.Engine(0)
    n = 256
    a_np = oracle.scaled_input(n, np.float32, 8)
    want = eng.power(a_np, 7)
    keep = []
    for i in range(80):
        a = torch.from_numpy(a_np).cuda()
        out = torch.empty_like(a)
        eng.power_device(a.data_ptr(), out.data_ptr(), n, 7)
        keep.append((a, out))
    eng.synchronize()
    for a, out in keep[::13]:
        assert out.cpu().numpy().tobytes() == want.tobytes()


def test_host_api_argument_validation(eng):
    with pytest.raises(ValueError):
        eng.power_mod(np.zeros(16, np.uint32), 3, 7)
    with pytest.raises(ValueError):
        eng.power_mod(np.zeros((4, 5), np.uint32), 3, 7)
    with pytest.raises(ValueError):
        eng.power_mod(np.zeros((4, 4), np.uint32), 3, 2**32 + 5)
    stack = np.zeros((3, 8, 8), np.float32)
    for bad in (np.zeros((2, 8, 8), np.float32), np.zeros((3, 8, 8), np.float64),
                np.zeros((3, 8, 16), np.float32)[:, :, ::2]):
        with pytest.raises(ValueError):
            eng.power_batched(stack, 3, out=bad)


def test_batched_host_api_pageable_equals_pinned(eng):
    """mxp_power_batched with ordinary (pageable) numpy arrays goes through the
    pinned staging ring; every combination of pageable / pinned input and
    output gives bitwise the same stack as the device path (several chunks,
    a ragged last chunk)."""
    n, batch, k = 128, 2 * 1024 + 333, 13
    stack = mx.scaled_batch(n, batch, mx.DType.F32, 17)
    want = eng.power_batched(stack, k)  # pageable in and out
    d_in, d_out = eng.alloc(stack.nbytes), eng.alloc(stack.nbytes)
    try:
        eng.upload(d_in, stack)
        eng.power_batched_device(d_in, d_out, n, batch, k)
        dev = np.empty_like(stack)
        eng.download(dev, d_out)
    finally:
        eng.free(d_in)
        eng.free(d_out)
    assert want.tobytes() == dev.tobytes()
    pin_in = eng.pinned_array(stack.shape, np.float32)
    pin_out = eng.pinned_array(stack.shape, np.float32)
    try:
        pin_in[...] = stack
        for src, dst in ((pin_in, pin_out), (pin_in, np.empty_like(stack)), (stack, pin_out)):
            dst[...] = 0
            eng.power_batched(src, k, out=dst)
            assert dst.tobytes() == want.tobytes()
            assert eng.last_stats.h2d_bytes == stack.nbytes == eng.last_stats.d2h_bytes
    finally:
        eng.host_free(pin_in.ctypes.data)
        eng.host_free(pin_out.ctypes.data)


def test_paper_table_with_b200_rows(capsys):
    """The paper's comparison table regenerated with B200 rows: repeated and
    squared on the b200 backend, merged with the reference CLI's own
    sequential-CPU rows (tests/golden/ref_naive_64.csv)."""
    import os

    from paper_1204_3052_b200 import cli

    ref_csv = os.path.join(os.path.dirname(__file__), "golden", "ref_naive_64.csv")
    assert cli.main(["bench", "--sizes", "64", "--powers", "2,16,64", "--reps", "2",
                     "--table", "-", "--baseline-csv", ref_csv]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "Matrix size 64 x 64"
    labels = ["Naïve GPU (In Sec)", "Sequential CPU (In Sec)", "Naïve Speed UP",
              "Our Approach (In Sec)", "Our Approach vs Naïve GPU"]
    assert [ln[:len(lab)] for ln, lab in zip(out[2:], labels)] == labels
    assert out[1].split() == ["2", "16", "64"]



@pytest.mark.parametrize("k,kernel", [(383, "k3h"), (384, "k3b")])
def test_router_threshold_both_kernels_meet_tolerance(eng, k, kernel):
    """Chains just below (K3H) and just above (K3B) the router's switch at
    n = 128: every matrix within the chain tolerance; the in-kernel clock
    stamps exist only after a K3H launch (which kernel really ran)."""
    n, batch = 128, 600
    assert _lib.small_kernel_for(n, k) == kernel
    stack = mx.scaled_batch(n, batch, mx.DType.F32, 31)
    d_in, d_out = eng.alloc(stack.nbytes), eng.alloc(stack.nbytes)
    try:
        eng.upload(d_in, stack)
        eng.power_batched_device(d_in, d_out, n, batch, k)
        out = np.empty_like(stack)
        eng.download(out, d_out)
        if kernel == "k3h":
            mhz, ms = eng.last_kernel_clock()
            assert 100 < mhz < 2500 and ms > 0
        else:
            with pytest.raises(mx.UnsupportedError):
                eng.last_kernel_clock()
    finally:
        eng.free(d_in)
        eng.free(d_out)
    ref = oracle.exponentiate_batched(stack, k, oracle.max_threads())
    tol = mx.fro_tol(n, k, "f32")
    for i in range(batch):
        assert fro(out[i], ref[i]) <= tol, (k, i, fro(out[i], ref[i]), tol)


@pytest.mark.parametrize("n", [64, 128, 384, 512, 1024])  # K3H, K3H, K1C, K1C, K1PH
def test_chain_strong_cancellation(eng, n):
    """A nilpotent-plus-small input: A = N + eps*R with N^2 = 0, so A^2 ~ eps
    and A^6 depends on entries ~eps^2 below the matrix max.  The 3xTF32
    chains keep an exponent per element; K3H's scaled fp16 planes keep one per
    matrix and would lose those entries (A^6 came out 50% wrong before the
    fixup, profiles/r02_cancellation_probe.txt), so K3H lists the matrix and
    K3B recomputes it.  Reference: the CPU fp32 chain's own distance from the
    exact result, with the reference's 64x device slack (tolerances.py:316-319)."""
    rng = np.random.default_rng(5)
    nil = np.zeros((n, n))
    nil[: n // 2, n // 2:] = rng.uniform(-1, 1, (n // 2, n // 2))
    a = (nil + 1e-6 * rng.uniform(-1, 1, (n, n))).astype(np.float32)
    bad = []
    for k in (2, 3, 6, 7):
        got = eng.power(a, k)
        if n <= 128 and k > 2:
            assert eng.last_small_fixups() == 1, (n, k)
        if n == 1024 and k > 2:
            assert eng.last_f32_fallback(), (n, k)
        ref = oracle.exponentiate(a, k, oracle.max_threads())
        exact = np.linalg.matrix_power(a.astype(np.float64), k)
        tol = max(mx.fro_tol_conditioned(n, k, "f32"), 64 * fro(ref, exact))
        if not fro(got, exact) <= tol:
            bad.append((k, fro(got, exact), fro(ref, exact), tol))
    assert not bad, (n, bad)


def test_small_n_fixup_inside_a_batch(eng):
    """Every 50th matrix of a random 128^2 batch is the cancelling construction:
    exactly those are recomputed, and every matrix meets its tolerance."""
    n, batch, k = 128, 600, 6
    stack = mx.scaled_batch(n, batch, mx.DType.F32, 77).astype(np.float64)
    rng = np.random.default_rng(9)
    special = list(range(3, batch, 50))
    for i in special:
        nil = np.zeros((n, n))
        nil[: n // 2, n // 2:] = rng.uniform(-1, 1, (n // 2, n // 2))
        stack[i] = nil + 1e-6 * rng.uniform(-1, 1, (n, n))
    stack = stack.astype(np.float32)
    d_in, d_out = eng.alloc(stack.nbytes), eng.alloc(stack.nbytes)
    try:
        eng.upload(d_in, stack)
        eng.power_batched_device(d_in, d_out, n, batch, k)
        out = np.empty_like(stack)
        eng.download(out, d_out)
        assert eng.last_small_fixups() == len(special)
        assert eng.last_stats.launches == 2
    finally:
        eng.free(d_in)
        eng.free(d_out)
    ref = oracle.exponentiate_batched(stack, k, oracle.max_threads())
    for i in range(batch):
        if i in special:
            exact = np.linalg.matrix_power(stack[i].astype(np.float64), k)
            tol = max(mx.fro_tol_conditioned(n, k, "f32"), 64 * fro(ref[i], exact))
            assert fro(out[i], exact) <= tol, (i, fro(out[i], exact), tol)
        else:
            assert fro(out[i], ref[i]) <= mx.fro_tol(n, k, "f32"), i


def test_one_launch_chain_zero_nan_identity(eng):
    """K1C edge inputs: a zero matrix, the identity to a high power (exact), and
    a NaN that must propagate where the reference's does."""
    z = np.zeros((512, 512), np.float32)
    assert not eng.power(z, 13).any()
    i = np.eye(300, dtype=np.float32)
    assert np.array_equal(eng.power(i, 1000), i)  # exact: powers of two only
    a = oracle.scaled_input(256, np.float32, 3)
    a[7, 9] = np.nan
    got = eng.power(a, 3)
    assert np.array_equal(np.isnan(got), np.isnan(oracle.exponentiate(a, 3)))



# ------------------------------------------------------------------ structured inputs, every kernel
def _structured(kind, n, rng):
    if kind == "upper_triangular":          # nilpotent strictly-upper part + a small diagonal
        a = np.triu(rng.uniform(-1, 1, (n, n)), 1) + np.diag(rng.uniform(-0.1, 0.1, n))
    elif kind == "two_scales":              # blocks 2^30 apart, coupled weakly
        a = rng.uniform(-1, 1, (n, n)) / np.sqrt(n)
        a[n // 2:, n // 2:] *= 2.0 ** -30
        a[: n // 2, n // 2:] *= 2.0 ** -15
    elif kind == "rank_one":                # u v^T: A^k = (v.u)^(k-1) A
        u, v = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        a = np.outer(u, v) / abs(v @ u)
    elif kind == "integer":                 # small integers: exact products while < 2^24
        a = rng.integers(-1, 2, (n, n)).astype(np.float64) * (rng.uniform(0, 1, (n, n)) < 2.0 / n)
    elif kind == "signed_permutation":
        p = rng.permutation(n)
        a = np.zeros((n, n))
        a[np.arange(n), p] = rng.choice([-1.5, 0.75], n)
    else:
        raise ValueError(kind)
    return a


@pytest.mark.parametrize("n,dt", [(64, "f32"), (128, "f32"), (300, "f32"), (1024, "f32"), (1600, "f32"),
                                  (256, "f64")])
@pytest.mark.parametrize("kind", ["upper_triangular", "two_scales", "rank_one", "integer",
                                  "signed_permutation"])
def test_structured_inputs_every_kernel(eng, n, dt, kind):
    """K3H/K3B (64, 128), K1C (300), K1PH (1024, and 1600 padded to 1792 whose
    3xTF32 recomputation runs on K1 at 1664) and K2 (f64): structured
    matrices with cancellation, wide dynamic range, low rank, exact integer
    products and permutations.  Criterion: no further from the exact result
    than the reference's own CPU chain by more than the reference's 64x
    device slack (tolerances.py:316-319), or inside the conditioned chain
    tolerance."""
    import zlib

    rng = np.random.default_rng(zlib.crc32(f"{kind}-{n}".encode()))
    npd = np.float32 if dt == "f32" else np.float64
    a = _structured(kind, n, rng).astype(npd)
    for k in (3, 8, 13):
        got = eng.power(a, k)
        ref = oracle.exponentiate(a, k, oracle.max_threads())
        exact = np.linalg.matrix_power(a.astype(np.float64), k)
        if not np.isfinite(exact).all():
            continue
        tol = max(mx.fro_tol_conditioned(n, k, dt), 64 * fro(ref, exact))
        assert np.array_equal(np.isfinite(got), np.isfinite(ref)), (kind, k)
        assert fro(got, exact) <= tol, (kind, n, k, fro(got, exact), fro(ref, exact), tol)
        if kind in ("integer", "signed_permutation") and np.abs(exact).max() < 2 ** 20:
            assert np.array_equal(got, exact.astype(npd)), (kind, k)  # exact arithmetic


def test_small_n_graph_survives_fixup_list_growth():
    """A cached n <= 128 chain graph holds the handle's fixup list; a batched
    launch larger than the list reallocates it, which must drop the graphs
    (a replay would otherwise write through a freed pointer)."""
    eng = mx.Engine(0)
    a = oracle.scaled_input(64, np.float32, 4)
    want = eng.power(a, 13)
    assert eng.power(a, 13).tobytes() == want.tobytes()  # cached graph
    big = mx.scaled_batch(64, 3000, mx.DType.F32, 1)  # > the initial 1024-entry list
    eng.power_batched(big, 13)
    for _ in range(3):
        assert eng.power(a, 13).tobytes() == want.tobytes()
    eng.synchronize()


def test_host_api_rejects_non_square_before_device_work():
    """Engine.multiply / power / power_mod validate shapes before the C call
    (a (5, 4) array would otherwise be read as 5 x 5)."""
    eng = mx.Engine(0)
    a = np.zeros((5, 4), np.float32)
    with pytest.raises(mx.ShapeError):
        eng.multiply(a, a)
    with pytest.raises(mx.ShapeError):
        eng.power(a, 3)
    with pytest.raises(mx.ShapeError):
        eng.power_mod(np.zeros((5, 4), np.uint32), 3, 97)
    with pytest.raises(mx.ShapeError):
        eng.multiply(np.zeros(16, np.float32), np.zeros(16, np.float32))
