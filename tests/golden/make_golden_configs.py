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
* c5: 8192x8192 f32 A^1024 (about 2-3 h on one core).

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
            res = single("c5", 8192, DType.F32, 1024)
        else:
            raise SystemExit(f"unknown config {name}")
        # re-read before writing: several invocations may run side by side
        try:
            with open(OUT) as fh:
                data = json.load(fh)
        except OSError:
            data = {}
        data[name] = res
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)
        print(name, res, flush=True)


if __name__ == "__main__":
    main()
