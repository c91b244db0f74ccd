"""C3 per-rank shard sizes on one GPU: time of one K3H launch over B matrices
(B = 65536 / N for N = 1, 2, 4, 8) — what each rank of an N-GPU strong-scaling
run does — and the implied scaling efficiency if the ranks ran in parallel."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1204_3052_b200 as mx  # noqa: E402

eng = mx.Engine(0)
w = bench.WORKLOADS["c3"]
base = None
for N in (1, 2, 4, 8, 16):
    B = 65536 // N
    ms, launches, clocks = bench.run_device(eng, w, 20, 3, 42, batch=B)
    if base is None:
        base = ms
    print(json.dumps({"N": N, "batch_per_rank": B, "ms": ms, "eff_vs_1": base / (N * ms),
                      "tflops_rank": bench.flops(w, B) / (ms / 1e3) / 1e12,
                      "sm_mhz_in_kernel": (clocks or {}).get("sm_mhz_in_kernel")}))
