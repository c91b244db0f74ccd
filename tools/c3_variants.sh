#!/bin/bash
# C3 (65536 x 128^2 A^64) device time with each library variant in tools/_variants/ and the product build, interleaved
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
for rep in 1 2 3; do
for lib in product tools/_variants/*.so; do
  if [ $lib = product ]; then unset MXP_LIB_PATH; else export MXP_LIB_PATH=$PWD/$lib; fi
  timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, paper_1204_3052_b200 as mx
eng = mx.Engine(0)
ms, l, c = bench.run_device(eng, bench.WORKLOADS['c3'], 20, 3, 42)
su = c.get('sustained', {})
print('$lib', f'{ms:.3f} ms', l, 'launches', f\"{c.get('sm_mhz_in_kernel', 0):.0f} MHz\", 'sustained', f\"{su.get('power_w') or 0:.0f} W\", f\"{su.get('sm_mhz_in_kernel') or 0:.0f} MHz\", su.get('reasons'))
" >> $O/c3_variants.txt 2>&1
done
done
unset MXP_LIB_PATH
