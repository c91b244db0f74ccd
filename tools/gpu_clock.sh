#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
nvidia-smi -q -d POWER,CLOCK > $O/smi_power.txt 2>&1
timeout 300 python tools/clock_check.py > $O/clock.txt 2>&1
