"""Hash of batched-power outputs (for bitwise A/B of kernel variants)."""
import hashlib
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx

eng = mx.Engine(0)
for n, B, k in ((128, 4096, 64), (128, 1200, 13), (100, 600, 257), (64, 800, 1000)):
    d_in = torch.empty((B, n, n), dtype=torch.float32, device="cuda")
    d_out = torch.empty_like(d_in)
    eng.random_device(d_in.data_ptr(), n, B, seed0=42, scale=math.sqrt(12.0 / n))
    eng.power_batched_device(d_in.data_ptr(), d_out.data_ptr(), n, B, k)
    eng.synchronize()
    h = hashlib.sha256(d_out.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"n={n} B={B} k={k} sha={h}")
