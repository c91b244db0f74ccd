"""Hashes of K1 chain / single-multiply / row-block outputs (bitwise A/B of
split-K variants: MXP_SPLITK=global vs the default cluster reduction)."""
import hashlib
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx

eng = mx.Engine(0)
h = lambda t: hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]
for n, k in ((130, 7), (200, 13), (256, 64), (384, 33), (512, 1000), (640, 5), (768, 3), (896, 9)):
    a = torch.empty((n, n), dtype=torch.float32, device="cuda")
    o = torch.empty_like(a)
    eng.random_device(a.data_ptr(), n, 1, seed0=42, scale=math.sqrt(12.0 / n))
    eng.power_device(a.data_ptr(), o.data_ptr(), n, k)
    eng.synchronize()
    line = f"n={n} k={k} chain={h(o)} launches={eng.last_stats.launches}"
    b = torch.empty_like(a)
    eng.random_device(b.data_ptr(), n, 1, seed0=7, scale=math.sqrt(12.0 / n))
    eng.gemm_device(a.data_ptr(), b.data_ptr(), o.data_ptr(), n)
    eng.synchronize()
    line += f" gemm={h(o)}"
    print(line, flush=True)
