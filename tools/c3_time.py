"""C3 launch timing (65536 x 128^2 A^64, inputs resident): median of reps."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx

n, k = 128, 64
B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
eng = mx.Engine(0)
d_in = torch.empty((B, n, n), dtype=torch.float32, device="cuda")
d_out = torch.empty_like(d_in)
eng.random_device(d_in.data_ptr(), n, B, seed0=42, scale=math.sqrt(12.0 / n))
for _ in range(3):
    eng.power_batched_device(d_in.data_ptr(), d_out.data_ptr(), n, B, k)
eng.synchronize()
s = torch.cuda.ExternalStream(eng.stream)
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.synchronize()
    e0.record(s)
    eng.power_batched_device(d_in.data_ptr(), d_out.data_ptr(), n, B, k)
    e1.record(s)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
fl = 2.0 * n ** 3 * 6 * B  # 6 multiplies for A^64
mean = sum(ts) / len(ts)
print(f"C3 B={B} median {ts[len(ts)//2]:.3f} ms mean {mean:.3f} min {ts[0]:.3f} -> {fl / ts[len(ts)//2] / 1e9:.1f} TFLOP/s")
