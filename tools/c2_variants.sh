#!/bin/bash
# C2 (512^2 A^1000, K1C) time + result hash with each library variant in tools/_variants/ and the product build
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
for rep in 1 2; do
for lib in product tools/_variants/*.so; do
  if [ $lib = product ]; then unset MXP_LIB_PATH; else export MXP_LIB_PATH=$PWD/$lib; fi
  timeout 300 python -c "
import sys, hashlib, numpy as np; sys.path.insert(0,'.')
import bench, oracle, paper_1204_3052_b200 as mx
eng = mx.Engine(0)
r = []
for _ in range(3):
    ms, l, _c = bench.run_device(eng, bench.WORKLOADS['c2'], 50, 5, 42, sample=False)
    r.append(ms * 1e3)
h = hashlib.sha256(eng.power(oracle.scaled_input(512, np.float32, 42), 1000).tobytes()).hexdigest()[:16]
print('$lib', ' '.join(f'{x:.1f}' for x in r), 'us', h)
" >> $O/c2_variants.txt 2>&1
done
done
unset MXP_LIB_PATH
