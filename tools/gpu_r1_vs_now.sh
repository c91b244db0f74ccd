#!/bin/bash
# C3 device time of the round-1 final build (tools/_variants/r1tree, af08815) and the current build, interleaved on one box
# (tools/_variants/r1tree: `git worktree add --detach tools/_variants/r1tree af08815`, then
#  build it in place with paper_1204_3052_b200.build; variants: tools/build_variant.py)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
for rep in 1 2 3 4; do
  (cd tools/_variants/r1tree && timeout 300 python tools/c3_time.py 65536 12 | sed 's/^/r1  /') >> $O/r1_vs_now.txt 2>&1
  timeout 300 python tools/c3_time.py 65536 12 | sed 's/^/now /' >> $O/r1_vs_now.txt 2>&1
done
nvidia-smi -q -d POWER,CLOCK > $O/smi_power.txt 2>&1
