"""Minimal C3 driver for ncu: device inputs, `reps` batched A^64 launches."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx

n, k = 128, int(sys.argv[2]) if len(sys.argv) > 2 else 64
B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
eng = mx.Engine(0)
d_in = torch.empty((B, n, n), dtype=torch.float32, device="cuda")
d_out = torch.empty_like(d_in)
eng.random_device(d_in.data_ptr(), n, B, seed0=42, scale=math.sqrt(12.0 / n))
for _ in range(2):
    eng.power_batched_device(d_in.data_ptr(), d_out.data_ptr(), n, B, k)
eng.synchronize()
print("ok")
