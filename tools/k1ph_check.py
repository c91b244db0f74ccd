"""K1PH (scaled fp16x2 large-n chain) vs the 3xTF32 chain and the oracle:
errors at a few sizes, the C5 step time both ways, and the fallback flag on a
cancelling input."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle
import paper_1204_3052_b200 as mx

eng = mx.Engine(0)
for n, k in ((1024, 13), (1536, 16), (2048, 7)):
    a = oracle.scaled_input(n, np.float32, 42)
    eng.set_f32_datapath("auto")
    g16 = eng.power(a, k)
    fb = eng.last_f32_fallback()
    eng.set_f32_datapath("3xtf32")
    g32 = eng.power(a, k)
    ref = oracle.exponentiate(a, k, oracle.max_threads())
    e16 = oracle.compare(g16, ref)[2]
    e32 = oracle.compare(g32, ref)[2]
    print(f"n={n} k={k}: fp16x2 {e16:.3e} (fallback {fb})  3xtf32 {e32:.3e}  tol {mx.fro_tol(n, k, 'f32'):.3e}", flush=True)

# cancelling input: N + 1e-6 R with N^2 = 0 (N = strictly block upper triangular)
n = 1024
rng = np.random.default_rng(3)
N = np.zeros((n, n), np.float32)
N[: n // 2, n // 2:] = rng.standard_normal((n // 2, n // 2)).astype(np.float32)
a = (N + 1e-6 * rng.standard_normal((n, n))).astype(np.float32)
eng.set_f32_datapath("auto")
g = eng.power(a, 6)
fb = eng.last_f32_fallback()
ref = oracle.exponentiate(a, 6, oracle.max_threads())
print(f"cancelling n={n} A^6: err {oracle.compare(g, ref)[2]:.3e} fallback {fb}", flush=True)

# C5 timing, inputs resident
n, k = 8192, 1024
d_in = torch.empty((n, n), dtype=torch.float32, device="cuda")
d_out = torch.empty_like(d_in)
eng.random_device(d_in.data_ptr(), n, 1, seed0=42, scale=(12.0 / n) ** 0.5)
s = torch.cuda.ExternalStream(eng.stream)
for dp in ("auto", "3xtf32", "auto"):
    eng.set_f32_datapath(dp)
    eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
    eng.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        eng.power_device(d_in.data_ptr(), d_out.data_ptr(), n, k)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"C5 {dp}: {ms:.2f} ms = {2 * n**3 * 10 / ms / 1e9:.1f} TFLOP/s", flush=True)
    if dp == "auto":
        print("  fallback", eng.last_f32_fallback())
