#!/bin/bash
# C3 launch time (tools/c3_time.py, synchronised launches): the round-1 build
# (tools/_variants/r1tree: `git worktree add --detach tools/_variants/r1tree af08815`, then
#  build it in place with paper_1204_3052_b200.build; variants: tools/build_variant.py)
# (tools/_variants/r1tree), the product, and every tools/_variants/*.so, interleaved
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
for rep in 1 2 3; do
  (cd tools/_variants/r1tree && timeout 300 python tools/c3_time.py 65536 12 | sed 's/^/r1 /') >> $O/k3h_ab.txt 2>&1
  for lib in product tools/_variants/*.so; do
    if [ $lib = product ]; then unset MXP_LIB_PATH; else export MXP_LIB_PATH=$PWD/$lib; fi
    timeout 300 python tools/c3_time.py 65536 12 | sed "s|^|$(basename $lib) |" >> $O/k3h_ab.txt 2>&1
  done
  unset MXP_LIB_PATH
done
