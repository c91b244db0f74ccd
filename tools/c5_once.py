"""One C5 chain (8192^2 A^1024) after a warm-up, inputs resident (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx

dp = sys.argv[1] if len(sys.argv) > 1 else "auto"
eng = mx.Engine(0)
eng.set_f32_datapath(dp)
n, k = 8192, 1024
d_in = torch.empty((n, n), dtype=torch.float32, device="cuda")
d_out = torch.empty_like(d_in)
eng.random_device(d_in.data_ptr(), n, 1, seed0=42, scale=(12.0 / n) ** 0.5)
for _ in range(2):
    eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
eng.synchronize()
print("done")
