"""C5 (8192^2 A^1024) chain time and a 2048^2 A^1024 error vs the oracle for
the library MXP_LIB_PATH points at (A/B of K1PH build variants)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle
import paper_1204_3052_b200 as mx

eng = mx.Engine(0)
tag = os.path.basename(os.environ.get("MXP_LIB_PATH", "product"))
a = oracle.scaled_input(2048, np.float32, 42)
err = oracle.compare(eng.power(a, 1024), oracle.exponentiate(a, 1024, oracle.max_threads()))[2]
n, k = 8192, 1024
d_in = torch.empty((n, n), dtype=torch.float32, device="cuda")
d_out = torch.empty_like(d_in)
eng.random_device(d_in.data_ptr(), n, 1, seed0=42, scale=(12.0 / n) ** 0.5)
s = torch.cuda.ExternalStream(eng.stream)
eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
eng.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
    e1.record(s)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{tag:16s} C5 median {ts[2]:.2f} ms min {ts[0]:.2f}  2048^2 A^1024 err {err:.3e}", flush=True)
