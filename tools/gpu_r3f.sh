#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 60 ./tools/k1c_trace 512 > $O/trace.txt 2>&1
