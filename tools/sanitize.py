"""Small invocations of every kernel family, for compute-sanitizer runs."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1204_3052_b200 as mx  # noqa: E402

eng = mx.Engine(0)
a = oracle.scaled_input(64, np.float32, 42)
eng.power(a, 13)                                   # K3H single chain (squares + base multiplies)
mx.exponentiate_batched(mx.scaled_batch(48, 300, mx.DType.F32, 1), 7)   # K3H batched, n < 128
mx.exponentiate_batched(mx.scaled_batch(37, 5, mx.DType.F32, 1), 5)    # K3H, n % 4 != 0
# K3H TMA IO path: n = 128, several matrices per chain, start-phase skew (batch >= 4 x 148)
mx.exponentiate_batched(mx.scaled_batch(128, 600, mx.DType.F32, 3), 13)
mx.exponentiate_batched(mx.scaled_batch(128, 300, mx.DType.F32, 3), 64)
mx.exponentiate_batched(mx.scaled_batch(128, 300, mx.DType.F32, 3), 1000)  # K3B via the bias guard
import torch  # noqa: E402
t = torch.from_numpy(oracle.random_matrix(512, np.float32, 9)).cuda()
o = torch.empty((128, 512), dtype=t.dtype, device=t.device)
eng.gemm_prepare_rhs_device(t.data_ptr(), 512)                          # prepared right-hand side
eng.gemm_rows_prepared_device(t[256:384].data_ptr(), o.data_ptr(), 512, 128)
eng.synchronize()
eng.power(oracle.scaled_input(384, np.float32, 42), 13)                 # K1C one-launch chain
eng.multiply(oracle.scaled_input(256, np.float32, 1), oracle.scaled_input(256, np.float32, 2))  # K1 cluster split-K
eng.power(oracle.scaled_input(1024, np.float32, 42), 5)                 # K1PH persistent pairs + split16
eng.power(oracle.scaled_input(1600, np.float32, 42), 3)                 # K1PH padded to 256 (1792)
nil = np.zeros((1024, 1024), np.float32)
nil[:512, 512:] = 1.0
eng.power((nil + np.float32(1e-6)).astype(np.float32), 6)                # K1PH flag -> gated 3xTF32 chain runs
print("k1ph fallback", eng.last_f32_fallback())
eng.set_f32_datapath("3xtf32")
eng.power(oracle.scaled_input(1024, np.float32, 42), 5)                 # K1P CTA pairs (3xTF32 datapath)
eng.set_f32_datapath("auto")
eng.power(oracle.scaled_input(256, np.float64, 42), 9)                  # FP64 DMMA
eng.power_mod(np.arange(100 * 100, dtype=np.uint32).reshape(100, 100), 11, 65521)  # K5I (INT8)
eng.power_mod(np.arange(300 * 300, dtype=np.uint32).reshape(300, 300) * 7919, 6, 2**31 - 1)
mx.random_matrix(33, mx.DType.F32, 5)
mx.splitmix64(42, 1000)
# K3H dynamic-range fixup: cancelling matrices inside a batch -> list-driven K3B pass
rng = np.random.default_rng(5)
stack = mx.scaled_batch(128, 300, mx.DType.F32, 3).astype(np.float64)
for i in (0, 150, 299):
    nil = np.zeros((128, 128))
    nil[:64, 64:] = rng.uniform(-1, 1, (64, 64))
    stack[i] = nil + 1e-6 * rng.uniform(-1, 1, (128, 128))
mx.exponentiate_batched(stack.astype(np.float32), 6)
print("fixups", mx.engine.default_engine(0).last_small_fixups())  # the engine exponentiate_batched used
# C2's shape: the one-launch K1C chain as a programmatic dependent of the split,
# grid-barrier counters reset by its last CTA (run twice: the second launch
# relies on the first one's reset)
eng.power(oracle.scaled_input(512, np.float32, 42), 1000)
eng.power(oracle.scaled_input(512, np.float32, 42), 1000)
# mxp_power_multi: batch shards, FP32 fused row shards, FP64 row shards (one GPU listed twice)
mx.exponentiate_multi(mx.scaled_batch(128, 300, mx.DType.F32, 3), 13, [0, 0])
mx.exponentiate_multi(oracle.scaled_input(1024, np.float32, 42), 5, [0, 0])
mx.exponentiate_multi(oracle.scaled_input(300, np.float64, 42), 5, [0, 0])
mx.engine.release_multi()
print("sanitize workload done")
