"""Cross-check K3H's in-kernel clock stamps (clock64 / globaltimer of CTA 0,
mxp_last_kernel_clock) against CUDA events around the same single launch."""
import math
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1204_3052_b200 as mx  # noqa: E402

eng = mx.Engine(0)
w = bench.WORKLOADS["c3"]
d_in, d_out, step = bench.device_workload(eng, w)
for _ in range(3):
    step()
eng.synchronize()
s = torch.cuda.ExternalStream(eng.stream)
for i in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    step()
    e1.record(s)
    e1.synchronize()
    mhz, kms = eng.last_kernel_clock()
    print(f"launch {i}: events {e0.elapsed_time(e1):.4f} ms, CTA0 globaltimer {kms:.4f} ms, "
          f"clock64/globaltimer {mhz:.0f} MHz, clock64/event-time {mhz * kms / e0.elapsed_time(e1):.0f} MHz",
          flush=True)
