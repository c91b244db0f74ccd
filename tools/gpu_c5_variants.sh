#!/bin/bash
# C5 chain time / accuracy of the product and every tools/_variants/k1ph*.so, interleaved
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
for rep in 1 2 3; do
  for lib in product tools/_variants/k1ph*.so; do
    if [ $lib = product ]; then unset MXP_LIB_PATH; else export MXP_LIB_PATH=$PWD/$lib; fi
    timeout 300 python tools/c5_variant.py >> $O/c5_variants.txt 2>&1
  done
  unset MXP_LIB_PATH
done
