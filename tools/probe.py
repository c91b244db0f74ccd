import sys, numpy as np, math
sys.path.insert(0, '.')
import oracle, paper_1204_3052_b200 as mx
what = sys.argv[1]
eng = mx.Engine(0)
if what == 'k3':
    for n,k in ((64,2),(64,16),(128,64),(48,13)):
        a = oracle.scaled_input(n, np.float32, 42)
        got = eng.power(a, k); ref = oracle.exponentiate(a, k)
        print('k3', n, k, oracle.compare(got, ref), mx.fro_tol(n,k,'f32'), flush=True)
elif what == 'k1':
    for n in (128, 256, 512):
        a = oracle.random_matrix(n, np.float32, 1); b = oracle.random_matrix(n, np.float32, 2)
        got = eng.multiply(a, b); ref = oracle.matmul(a, b)
        print('k1mul', n, oracle.compare(got, ref), n*2**-24*64, flush=True)
    a = oracle.scaled_input(512, np.float32, 42)
    got = eng.power(a, 1000); ref = oracle.exponentiate(a, 1000)
    print('k1chain', oracle.compare(got, ref), mx.fro_tol(512,1000,'f32'), flush=True)
elif what == 'f64':
    for n in (64, 256):
        a = oracle.random_matrix(n, np.float64, 1); b = oracle.random_matrix(n, np.float64, 2)
        got = eng.multiply(a, b); ref = oracle.matmul(a, b)
        print('f64mul', n, oracle.compare(got, ref), flush=True)
elif what == 'gen':
    print(mx.random_matrix(2, mx.DType.F64, 42).array.ravel().tolist())
if what == 'diag':
    n = 128
    I = np.eye(n, dtype=np.float32)
    rr = np.repeat(np.arange(n, dtype=np.float32)[:, None], n, 1)
    rc = rr.T.copy()
    for name, a, b in (("I*Rrow", I, rr), ("I*Rcol", I, rc), ("Rrow*I", rr, I), ("Rcol*I", rc, I)):
        got = eng.multiply(a, b); ref = a @ b
        ok = np.array_equal(got, ref)
        print(name, 'ok' if ok else 'BAD', flush=True)
        if not ok:
            np.save(f'gpurun_out/diag_{name.replace("*","_")}.npy', got)
            print(got[:4, :8]); print(got[32:34, :8]); print(got[:4, 32:40])
if what == 'acc':
    for n in (128, 512, 2048):
        a = oracle.random_matrix(n, np.float32, 1); b = oracle.random_matrix(n, np.float32, 2)
        exact = a.astype(np.float64) @ b.astype(np.float64)
        cpu = oracle.matmul(a, b)
        got = eng.multiply(a, b)
        # tf32-exact inputs: lo == 0, only hi*hi products (exact) -> pure accumulation error
        at = (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
        bt = (b.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
        exact_t = at.astype(np.float64) @ bt.astype(np.float64)
        got_t = eng.multiply(at, bt)
        cpu_t = oracle.matmul(at, bt)
        f = lambda x, r: oracle.compare(x, r)[2]
        bias = lambda x, r: float(np.mean((np.abs(x.astype(np.float64)) - np.abs(r)) / (np.abs(r).mean())))
        print(f"n={n} fro vs exact: cpu {f(cpu, exact):.3e} tc {f(got, exact):.3e} | tf32-exact inputs: cpu {f(cpu_t, exact_t):.3e} tc {f(got_t, exact_t):.3e} | tc mean(|x|-|r|)/|r| {bias(got_t, exact_t):.2e} cpu {bias(cpu_t, exact_t):.2e}", flush=True)
