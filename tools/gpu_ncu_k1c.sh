#!/bin/bash
# ncu --set full of C2's one-launch chain (K1C) on the current build
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1c_chain -c 1 \
  -o $O/prof_k1c -f python tools/c2_once.py c2 2 > $O/ncu_k1c.log 2>&1
echo "rc=$?" >> $O/ncu_k1c.log
