#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 120 ./tools/gridbar_probe > $O/gridbar.txt 2>&1
