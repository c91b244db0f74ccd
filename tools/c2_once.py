"""One chain of a bench workload (default C2, 512^2 A^1000) through the
bench's device path, a few times; prints the result hash (for ncu runs of
the one-launch K1C chain)."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1204_3052_b200 as mx  # noqa: E402

eng = mx.Engine(0)
w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
d_in, d_out, step = bench.device_workload(eng, w)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    step()
eng.synchronize()
out = np.empty((w["n"], w["n"]), np.float32 if w["dtype"] == "f32" else np.float64)
eng.download(out, d_out)
print("hash", hashlib.sha256(out.tobytes()).hexdigest()[:16], "launches", eng.last_stats.launches)
