#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2u; mkdir -p $O
timeout 120 ./tools/i8_probe > $O/i8_probe.txt 2>&1; echo "rc=$?" >> $O/i8_probe.txt
