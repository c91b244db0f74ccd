"""C4-shaped FP64 chain timing (4096^2 A^257 by default; graph replay)."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx
from paper_1204_3052_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
k = int(sys.argv[2]) if len(sys.argv) > 2 else 257
eng = mx.Engine(0)
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
o = torch.empty_like(a)
eng.random_device(a.data_ptr(), n, 1, seed0=42, scale=math.sqrt(12.0 / n), mode=_lib.MXP_F64)
for _ in range(2):
    eng.power_device(a.data_ptr(), o.data_ptr(), n, k, mode=_lib.MXP_F64)
eng.synchronize()
s = torch.cuda.ExternalStream(eng.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(3):
    eng.power_device(a.data_ptr(), o.data_ptr(), n, k, mode=_lib.MXP_F64)
e1.record(s)
e1.synchronize()
ms = e0.elapsed_time(e1) / 3
m = bin(k).count("1") + k.bit_length() - 2
print(f"f64 n={n} k={k}: {ms:.2f} ms  {2 * n ** 3 * m / ms / 1e9:.1f} TFLOP/s")
