#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2i; mkdir -p $O
timeout 120 python tools/mc_probe.py > $O/mc_probe.txt 2>&1; echo "rc=$?" >> $O/mc_probe.txt
ls /dev/nvidia* >> $O/mc_probe.txt 2>&1; (nvidia-smi -q | grep -i -A3 "fabric\|imex") >> $O/mc_probe.txt 2>&1
