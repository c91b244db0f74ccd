#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
for rep in 1 2; do
for lib in product tools/_variants/*.so; do
  if [ $lib = product ]; then unset MXP_LIB_PATH; else export MXP_LIB_PATH=$PWD/$lib; fi
  timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, paper_1204_3052_b200 as mx
eng = mx.Engine(0)
r = []
for _ in range(3):
    ms, l, _c = bench.run_device(eng, bench.WORKLOADS['c1'], 200, 20, 42, sample=False)
    r.append(ms * 1e3)
print('$lib', ' '.join(f'{x:.2f}' for x in r), 'us', l, 'launches')
" >> $O/c1_variants.txt 2>&1
done
done
