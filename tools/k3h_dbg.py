import sys, math, numpy as np
sys.path.insert(0, ".")
import oracle, paper_1204_3052_b200 as mx
for n, batch, k in ((128, 1, 64), (128, 149, 7), (128, 297, 2), (128, 300, 64), (128, 600, 64), (128, 1200, 13), (64, 600, 64)):
    stack = mx.scaled_batch(n, batch, mx.DType.F32, 21)
    try:
        out = mx.exponentiate_batched(stack, k)
        bad = [i for i in range(batch) if not np.isfinite(out[i]).all() or oracle.compare(out[i], oracle.exponentiate(stack[i], k))[2] > mx.fro_tol(n, k, "f32")] if batch <= 300 else [i for i in (0, 1, batch//2, batch-1) if not np.isfinite(out[i]).all()]
        print(n, batch, k, "bad", len(bad), bad[:10], flush=True)
    except Exception as e:
        print(n, batch, k, "EXC", e, flush=True); break
