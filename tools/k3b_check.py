"""K3 variant check on the GPU: accuracy vs the oracle / exact f64 and C3 time.

    MXP_K3=tf32 python tools/k3b_check.py    # 3xTF32 single-chain K3
    python tools/k3b_check.py                # bf16x3 dual-chain K3B
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # checker only
import paper_1204_3052_b200 as mx

tag = os.environ.get("MXP_K3", "k3b")
eng = mx.Engine(0)
torch.cuda.set_device(0)

# --- accuracy: single matrices through the host API
for n, k in ((64, 16), (128, 64), (48, 13), (128, 1000), (100, 257), (7, 3), (128, 2)):
    a = oracle.scaled_input(n, np.float32, 42)
    got = eng.power(a, k)
    ref = oracle.exponentiate(a, k)
    exact = np.linalg.matrix_power(a.astype(np.float64), k)
    e_ref = oracle.compare(got, ref)[2]
    e_ex = oracle.compare(got, exact)[2]
    e_cpu = oracle.compare(ref, exact)[2]
    print(f"[{tag}] n={n:3d} k={k:4d} fro vs oracle {e_ref:.3e} vs exact {e_ex:.3e} "
          f"(cpu fp32 vs exact {e_cpu:.3e}) tol {mx.fro_tol(n, k, 'f32'):.2e}", flush=True)

# single multiply accuracy / bias (k = 2 on random inputs)
a = oracle.random_matrix(128, np.float32, 1)
got = eng.power(a, 2)
exact = a.astype(np.float64) @ a.astype(np.float64)
bias = float(np.mean((np.abs(got.astype(np.float64)) - np.abs(exact))) / np.abs(exact).mean())
print(f"[{tag}] A^2 n=128 fro vs exact {oracle.compare(got, exact)[2]:.3e} bias {bias:.2e}", flush=True)

# --- batched: C3 shape, a few matrices checked against the oracle
n, k, B = 128, 64, 65536
d_in = torch.empty((B, n, n), dtype=torch.float32, device="cuda")
d_out = torch.empty_like(d_in)
eng.random_device(d_in.data_ptr(), n, B, seed0=42, scale=math.sqrt(12.0 / n))
eng.power_batched_device(d_in.data_ptr(), d_out.data_ptr(), n, B, k)
eng.synchronize()
worst = 0.0
for i in (0, 1, 147, 148, 149, 295, 296, 4097, 65535):
    a = d_in[i].cpu().numpy()
    worst = max(worst, oracle.compare(d_out[i].cpu().numpy(), oracle.exponentiate(a, k))[2])
print(f"[{tag}] C3 sample worst fro vs oracle {worst:.3e} tol {mx.fro_tol(n, k, 'f32'):.2e}", flush=True)
st = torch.cuda.Stream(torch.device("cuda", 0))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    eng.power_batched_device(d_in.data_ptr(), d_out.data_ptr(), n, B, k)
eng.synchronize()
times = []
s = torch.cuda.ExternalStream(eng.stream)
for _ in range(10):
    ev0.record(s)
    eng.power_batched_device(d_in.data_ptr(), d_out.data_ptr(), n, B, k)
    ev1.record(s)
    ev1.synchronize()
    times.append(ev0.elapsed_time(ev1))
ms = float(np.median(times))
fl = 2.0 * n ** 3 * 6 * B
print(f"[{tag}] C3 {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s  (min {min(times):.3f})", flush=True)
# odd sizes / multiply-heavy plans in batch
for n, k, B in ((128, 1000, 4096), (96, 13, 1000), (33, 7, 300)):
    d_in = torch.empty((B, n, n), dtype=torch.float32, device="cuda")
    d_out = torch.empty_like(d_in)
    eng.random_device(d_in.data_ptr(), n, B, seed0=7, scale=math.sqrt(12.0 / n))
    eng.power_batched_device(d_in.data_ptr(), d_out.data_ptr(), n, B, k)
    eng.synchronize()
    worst = 0.0
    for i in (0, 1, B // 2, B - 1):
        a = d_in[i].cpu().numpy()
        worst = max(worst, oracle.compare(d_out[i].cpu().numpy(), oracle.exponentiate(a, k))[2])
    print(f"[{tag}] batch n={n} k={k} B={B} worst fro {worst:.3e} tol {mx.fro_tol(n, k, 'f32'):.2e}",
          flush=True)
