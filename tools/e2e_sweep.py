"""e2e (host API, pinned buffers) time of the C3 batch for the built chunk size."""
import sys, time, math, statistics
import numpy as np
sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx
eng = mx.Engine(0)
n, B, k = 128, 65536, 64
hin = eng.pinned_array((B, n, n), np.float32); hout = eng.pinned_array((B, n, n), np.float32)
d = eng.alloc(hin.nbytes); eng.random_device(d, n, B, 42, -0.5, 0.5, math.sqrt(12 / n)); eng.download(hin, d); eng.free(d)
eng.power_batched(hin, k, out=hout)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); eng.power_batched(hin, k, out=hout); ts.append(time.perf_counter() - t0)
med = statistics.median(ts)
print(f"e2e {med*1e3:.1f} ms  {2*n**3*6*B/med/1e12:.1f} TFLOP/s  device {eng.last_stats.device_ms:.1f} ms")
