"""Pin the oracle at the BASELINE config sizes with the UNMODIFIED reference
(run in the build container only; /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_configs.py [c3] [c4] [c5]

For each config the reference's own public API computes the full result
(`exponentiate(A, k, naive_backend())`, expo.py:121-139, whose multiply is
`matmul_naive`, linalg.py:151-164) on the SURVEY §8(d) input recipe, and the
sha256 of the result bytes goes into tests/golden/configs.json:

* c3: all 65536 matrices of 128x128 f32 A^64 (seeds 42+i), hashed as one
      (65536, 128, 128) stack.  Independent matrices, so a process pool runs
      whole reference chains in parallel (each chain is the reference's own
      single-threaded call).
* c4: 4096x4096 f64 A^257 (about 20 min on one core).
* c5: 8192x8192 f32 A^1024.  One core would take ~5 h, so the reference's
      own `exponentiate` (plan, step order, accumulator on the left) drives
      a backend that applies `matmul_naive`'s loop body
      (c += a[:, k, None] * b[None, k, :], ascending k, linalg.py:151-164)
      to row blocks in worker processes.  Every element is the same scalar
      sequence fl(c + fl(a_ik * b_kj)) whatever the row blocking, so the
      result is bitwise the unmodified call's; the script first checks that
      against the unmodified `matmul_naive` on 512^2 / 1024^2 products
      (`c5_rowpar` records the check).

tests/test_gpu_parity.py recomputes the same results with the C oracle on
the GPU box, asserts that they hash to these reference values (so the oracle
is pinned at full size, not only on small fixtures), and then checks the
device results against them.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from matexpo import DType, Matrix, exponentiate, naive_backend, random_matrix  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "configs.json")


def scaled(n: int, dtype: DType, seed: int) -> Matrix:
    s = math.sqrt(12.0 / n)
    return Matrix((random_matrix(n, DType.F64, seed).array * s).astype(dtype.np))


def _c3_chunk(args):
    lo, hi = args
    out = np.empty((hi - lo, 128, 128), dtype=np.float32)
    for i in range(lo, hi):
        out[i - lo] = exponentiate(scaled(128, DType.F32, 42 + i), 64, naive_backend()).array
    return lo, out.tobytes()


def c3(workers: int) -> dict:
    batch, chunk = 65536, 512
    h = hashlib.sha256()
    parts = {}
    t0 = time.time()
    with ProcessPoolExecutor(workers) as pool:
        for lo, blob in pool.map(_c3_chunk, [(i, min(i + chunk, batch))
                                             for i in range(0, batch, chunk)]):
            parts[lo] = blob
    for lo in sorted(parts):
        h.update(parts[lo])
    return {"config": "c3: 65536 x 128x128 f32 A^64, seeds 42+i, scaled recipe",
            "sha256_stack": h.hexdigest(), "seconds": time.time() - t0, "workers": workers}


_SH = {}


def _attach(names):
    from multiprocessing import shared_memory
    for nm in names:
        if nm not in _SH:
            _SH[nm] = shared_memory.SharedMemory(name=nm)
    return _SH


def _rows_job(args):
    """matmul_naive's loop body (linalg.py:159-161) on rows [r0, r1), 32 rows
    at a time (the block stays in cache); per element the same ascending-k
    sequence of rounded products and rounded adds as the unmodified call."""
    a_nm, b_nm, c_nm, n, r0, r1 = args
    sh = _attach((a_nm, b_nm, c_nm))
    a = np.ndarray((n, n), np.float32, buffer=sh[a_nm].buf)
    b = np.ndarray((n, n), np.float32, buffer=sh[b_nm].buf)
    c = np.ndarray((n, n), np.float32, buffer=sh[c_nm].buf)
    for lo in range(r0, r1, 32):
        hi = min(lo + 32, r1)
        blk = np.zeros((hi - lo, n), np.float32)
        av = a[lo:hi]
        for k in range(n):
            blk += av[:, k, None] * b[None, k, :]
        c[lo:hi] = blk
    return r0


class RowParallelNaive:
    """A backend multiply equal bit for bit to matmul_naive, run on row blocks
    in a process pool over shared memory (f32 only)."""

    def __init__(self, n: int, workers: int):
        from multiprocessing import shared_memory
        self.n, self.workers = n, workers
        self.shm = [shared_memory.SharedMemory(create=True, size=n * n * 4) for _ in range(3)]
        self.pool = ProcessPoolExecutor(workers)

    def _arr(self, i):
        return np.ndarray((self.n, self.n), np.float32, buffer=self.shm[i].buf)

    def multiply(self, a: Matrix, b: Matrix) -> Matrix:
        n = self.n
        assert a.n == n and b.n == n and a.array.dtype == np.float32
        self._arr(0)[...] = a.array
        self._arr(1)[...] = b.array
        step = -(-n // (4 * self.workers))
        jobs = [(self.shm[0].name, self.shm[1].name, self.shm[2].name, n, r, min(r + step, n))
                for r in range(0, n, step)]
        list(self.pool.map(_rows_job, jobs))
        return Matrix(self._arr(2).copy(), copy=False)

    def close(self):
        self.pool.shutdown()
        for s in self.shm:
            s.close()
            s.unlink()


def rowpar_check(workers: int) -> list:
    from matexpo import matmul_naive
    done = []
    for n in (512, 1024):
        a, b = scaled(n, DType.F32, 7), scaled(n, DType.F32, 8)
        rp = RowParallelNaive(n, workers)
        try:
            got = rp.multiply(a, b).array
        finally:
            rp.close()
        ref = matmul_naive(a, b).array
        if got.tobytes() != ref.tobytes():
            raise SystemExit(f"row-parallel multiply differs from matmul_naive at n={n}")
        done.append(n)
    return done


def c5_rowpar(workers: int) -> dict:
    from matexpo import Backend
    checked = rowpar_check(workers)
    t0 = time.time()
    rp = RowParallelNaive(8192, workers)
    try:
        r = exponentiate(scaled(8192, DType.F32, 42), 1024, Backend("naive-rowpar", rp.multiply)).array
    finally:
        rp.close()
    return {"config": "c5: 8192x8192 f32 A^1024, seed 42, scaled recipe",
            "sha256": hashlib.sha256(np.ascontiguousarray(r).tobytes()).hexdigest(),
            "seconds": time.time() - t0, "workers": workers,
            "method": "reference exponentiate + matmul_naive loop body on row blocks "
                      f"(bitwise-checked against matmul_naive at n={checked})"}


def single(name: str, n: int, dt: DType, k: int) -> dict:
    t0 = time.time()
    r = exponentiate(scaled(n, dt, 42), k, naive_backend()).array
    return {"config": f"{name}: {n}x{n} {dt.name.lower()} A^{k}, seed 42, scaled recipe",
            "sha256": hashlib.sha256(np.ascontiguousarray(r).tobytes()).hexdigest(),
            "seconds": time.time() - t0, "workers": 1}


def main() -> None:
    which = sys.argv[1:] or ["c3", "c4", "c5"]
    try:
        with open(OUT) as fh:
            data = json.load(fh)
    except OSError:
        data = {}
    for name in which:
        if name == "c3":
            res = c3(int(os.environ.get("C3_WORKERS", "6")))
        elif name == "c4":
            res = single("c4", 4096, DType.F64, 257)
        elif name == "c5":
            res = c5_rowpar(int(os.environ.get("C5_WORKERS", "7")))
        elif name == "c5_single":  # the unmodified one-core call (~5 h)
            res = single("c5", 8192, DType.F32, 1024)
        else:
            raise SystemExit(f"unknown config {name}")
        # re-read before writing: several invocations may run side by side
        try:
            with open(OUT) as fh:
                data = json.load(fh)
        except OSError:
            data = {}
        data["c5" if name == "c5_single" and "c5" not in data else name] = res
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
        print(name, res, flush=True)


if __name__ == "__main__":
    main()
