#!/bin/bash
# run one probe binary: gpu_probe.sh <out-subdir> <binary> [args]
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O; shift
nvidia-smi --query-gpu=power.limit,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 300 "$@" > $O/out.txt 2>&1; echo "rc=$?" >> $O/out.txt
