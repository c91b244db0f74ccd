"""Generate tests/golden/ from the UNMODIFIED reference (run in the build
container only; /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every value below is produced by calling the reference's own public API
(`matexpo.splitmix64`, `random_matrix`, `exponentiate`, `naive_backend`,
`repeated_exponentiate`); nothing is recomputed locally.  The oracle
(oracle/) is then pinned bit-for-bit against these fixtures by
tests/test_oracle.py, and the GPU parity tests compare against the same
fixtures within tolerance.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import matexpo  # noqa: E402
from matexpo import (  # noqa: E402
    DType,
    Matrix,
    exponentiate,
    naive_backend,
    random_matrix,
    repeated_exponentiate,
    splitmix64,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def scaled(n: int, dtype: DType, seed: int) -> Matrix:
    """SURVEY §8(d) recipe, built from the reference generator."""
    s = math.sqrt(12.0 / n)
    return Matrix((random_matrix(n, DType.F64, seed).array * s).astype(dtype.np))


def main() -> None:
    t0 = time.time()
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": "matexpo " + matexpo.__version__, "entries": {}}

    # 1. SplitMix64 streams (test_linalg.py:28-45 pins the first 4).
    for seed in (0, 42, 2024, 7, 2**64 - 1):
        arrays[f"sm64_{seed}"] = splitmix64(seed, 16)

    # 2. random_matrix (linalg.py:127-148), incl. the frozen KATs.
    rm_cases = [(2, "f64", 42, -0.5, 0.5), (4, "f32", 7, -0.5, 0.5), (8, "f32", 3, -0.5, 0.5),
                (33, "f64", 5, -0.5, 0.5), (16, "f32", 9, -100.0, 100.0),
                (16, "f32", 42, -0.025, 0.025), (5, "f64", 11, 2.0, 3.0)]
    for n, dt, seed, lo, hi in rm_cases:
        key = f"rm_{n}_{dt}_{seed}_{lo}_{hi}"
        arrays[key] = random_matrix(n, DType.parse(dt), seed, lo, hi).array
    big_rm = {}
    for n, dt, seed in [(128, "f32", 42), (512, "f64", 42), (1024, "f32", 43)]:
        big_rm[f"{n}_{dt}_{seed}"] = sha(random_matrix(n, DType.parse(dt), seed).array)
    meta["random_matrix_sha256"] = big_rm

    # 3. Scaled inputs (the configs' recipe) — hashes of the exact bits.
    meta["scaled_sha256"] = {
        f"{n}_{dt}_{seed}": sha(scaled(n, DType.parse(dt), seed).array)
        for n, dt, seed in [(64, "f32", 42), (128, "f32", 42), (128, "f32", 43),
                            (512, "f32", 42), (256, "f64", 42)]
    }

    # 4. exponentiate on the naive backend (expo.py:121-139): full arrays.
    powers = (0, 1, 2, 3, 7, 13, 16, 64)
    for dt in ("f32", "f64"):
        for n in (2, 4, 8, 16, 64):
            a = scaled(n, DType.parse(dt), 42)
            arrays[f"in_{n}_{dt}"] = a.array
            for k in powers:
                arrays[f"exp_{n}_{dt}_{k}"] = exponentiate(a, k, naive_backend()).array

    # 4b. the reference's own default (unscaled) input for config 1.
    a = random_matrix(64, DType.F32, 42)
    arrays["unscaled_in_64_f32"] = a.array
    arrays["unscaled_exp_64_f32_16"] = exponentiate(a, 16, naive_backend()).array

    # 4c. host.test.ts:173-184 well-conditioned input (0.9 I + U[-0.025,0.025)).
    noise = random_matrix(64, DType.F32, 42, -0.025, 0.025).array.copy()
    noise[np.arange(64), np.arange(64)] += np.float32(0.9)
    wc = Matrix(noise)
    arrays["wc_in_64_f32"] = wc.array
    arrays["wc_exp_64_f32_64"] = exponentiate(wc, 64, naive_backend()).array
    arrays["wc_rep64_64_f64"] = repeated_exponentiate(wc.astype(DType.F64), 64,
                                                     naive_backend()).array

    # 4d. F64 repeated oracle on the oracle grid (test_acceptance.py:132-152).
    for n in (2, 4, 8, 16):
        base = random_matrix(n, DType.F64, 42)
        for k in (1, 2, 3, 7, 13, 64):
            arrays[f"rep_{n}_f64_{k}"] = repeated_exponentiate(base, k, naive_backend()).array

    # 5. Fibonacci Q^10 (test_expo.py:113-117) and Q^k for larger exact k.
    q = Matrix.from_rows([[1.0, 1.0], [1.0, 0.0]], DType.F64)
    for k in (10, 40, 78):
        arrays[f"fib_f64_{k}"] = exponentiate(q, k, naive_backend()).array

    # 6. Config C3 samples: 128x128 f32 A^64, batch element i has seed 42+i.
    c3 = {}
    for i in (0, 1, 255, 4097, 65535):
        r = exponentiate(scaled(128, DType.F32, 42 + i), 64, naive_backend()).array
        c3[str(i)] = sha(r)
        if i in (0, 65535):
            arrays[f"c3_out_{i}"] = r
    meta["c3_exp_sha256"] = c3

    # 7. Config C2: 512x512 f32 A^1000 (14 multiplies) and A^16 at 256/512.
    meta["c2_exp_sha256"] = sha(exponentiate(scaled(512, DType.F32, 42), 1000,
                                             naive_backend()).array)
    meta["exp_256_f32_16_sha256"] = sha(exponentiate(scaled(256, DType.F32, 42), 16,
                                                     naive_backend()).array)
    meta["exp_256_f64_257_sha256"] = sha(exponentiate(scaled(256, DType.F64, 42), 257,
                                                      naive_backend()).array)
    # one reference multiply at a non-tile size (ragged edges)
    a = random_matrix(200, DType.F32, 5)
    b = random_matrix(200, DType.F32, 6)
    meta["mm_200_f32_sha256"] = sha(matexpo.matmul_naive(a, b).array)
    arrays["exp_100_f32_13"] = exponentiate(scaled(100, DType.F32, 42), 13,
                                            naive_backend()).array
    # row-stochastic 5x5 (spectral radius exactly 1): A^1000 stays finite
    st = random_matrix(5, DType.F32, 42, 0.0, 1.0).array
    st = (st / st.sum(axis=1, keepdims=True)).astype(np.float32)
    arrays["stoch_in_5_f32"] = st
    arrays["stoch_exp_5_f32_1000"] = exponentiate(Matrix(st), 1000, naive_backend()).array

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
