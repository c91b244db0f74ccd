"""C1-shaped single small chains (one K3H CTA): device time vs plan length,
separating the fixed cost (graph launch, prologue, load/store, the fixup
pass) from the per-step cost."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx  # noqa: E402

eng = mx.Engine(0)
for n in (64, 128):
    d_in = torch.empty((n, n), dtype=torch.float32, device="cuda")
    d_out = torch.empty_like(d_in)
    eng.random_device(d_in.data_ptr(), n, 1, seed0=42, scale=math.sqrt(12.0 / n))
    for k in (2, 4, 16, 256, 2**12):
        for _ in range(5):
            eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
        eng.synchronize()
        s = torch.cuda.ExternalStream(eng.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(50):
            eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
        e1.record(s)
        e1.synchronize()
        steps = k.bit_length() - 1 + bin(k).count("1") - 1
        print(f"n={n} k={k} steps={steps}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us "
              f"({mx.engine._lib.load() and eng.last_stats.launches} launches)", flush=True)
