"""C2 (512^2 A^1000) and C5 (8192^2 A^1024) device-chain timing (graph replay)."""
import sys, math
import torch
sys.path.insert(0, ".")
import paper_1204_3052_b200 as mx
eng = mx.Engine(0)
for n, k, reps in ((512, 1000, 50), (1024, 1000, 20), (8192, 1024, 3)):
    d_in = torch.empty((n, n), dtype=torch.float32, device="cuda"); d_out = torch.empty_like(d_in)
    eng.random_device(d_in.data_ptr(), n, 1, seed0=42, scale=math.sqrt(12.0 / n))
    for _ in range(3): eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
    eng.synchronize()
    s = torch.cuda.ExternalStream(eng.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps): eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
    e1.record(s); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    m = bin(k).count("1") + k.bit_length() - 2
    print(f"n={n} k={k}: {ms*1e3:.1f} us  {2*n**3*m/ms/1e9:.1f} TFLOP/s  launches {eng.last_stats.launches}", flush=True)
