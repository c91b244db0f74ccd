#!/bin/bash
# run one python tool on the box: gpu_misc.sh <out-subdir> <script> [args]
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O; shift
timeout 900 python "$@" > $O/out.txt 2>&1; echo "rc=$?" >> $O/out.txt
