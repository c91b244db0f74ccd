#!/bin/bash
# C5 (8192^2 A^1024, K1P chain) time + result hash with the product build and each tools/_variants/*.so
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
for rep in 1 2; do
for lib in product tools/_variants/*.so; do
  if [ $lib = product ]; then unset MXP_LIB_PATH; else export MXP_LIB_PATH=$PWD/$lib; fi
  timeout 300 python -c "
import sys, hashlib, numpy as np; sys.path.insert(0,'.')
import bench, paper_1204_3052_b200 as mx
eng = mx.Engine(0)
w = bench.WORKLOADS['c5']
r = []
for _ in range(3):
    ms, l, _c = bench.run_device(eng, w, 10, 3, 42, sample=False)
    r.append(ms)
d_in, d_out, step = bench.device_workload(eng, w)
step(); eng.synchronize()
out = np.empty((w['n'], w['n']), np.float32); eng.download(out, d_out)
print('$lib', ' '.join(f'{x:.3f}' for x in r), 'ms', l, 'launches', hashlib.sha256(out.tobytes()).hexdigest()[:16])
" >> $O/c5_variants.txt 2>&1
done
done
unset MXP_LIB_PATH
