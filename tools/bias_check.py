"""Per-multiply bias of the small-n kernels vs n (A^2 of random inputs, exact f64 reference)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # checker only
import paper_1204_3052_b200 as mx

tag = "k3h/k3b (as routed)"
eng = mx.Engine(0)
for n in (8, 16, 32, 48, 64, 96, 128):
    biases, errs = [], []
    for seed in range(1, 9):
        a = oracle.random_matrix(n, np.float32, seed)
        got = eng.power(a, 2).astype(np.float64)
        exact = a.astype(np.float64) @ a.astype(np.float64)
        biases.append(float(np.mean(np.abs(got) - np.abs(exact)) / np.abs(exact).mean()))
        errs.append(oracle.compare(got, exact)[2])
    print(f"[{tag}] n={n:3d} bias {np.mean(biases):+.3e}  fro {np.mean(errs):.3e}", flush=True)
