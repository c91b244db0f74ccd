#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2m; mkdir -p $O
timeout 300 python tools/pcie_streams_probe.py > $O/pcie_streams.txt 2>&1
timeout 300 python tools/pcie_probe.py >> $O/pcie_streams.txt 2>&1
