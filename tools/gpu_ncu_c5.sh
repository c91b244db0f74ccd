#!/bin/bash
# C5 launch list (K1PH chain) and one full ncu capture of a K1PH GEMM step
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c5_launches.csv python tools/c5_once.py > $O/c5_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1ph -s 12 -c 1 -o $O/k1ph_full python tools/c5_once.py > $O/k1ph_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:split16 -s 12 -c 1 -o $O/split16_full python tools/c5_once.py > $O/split16_full.log 2>&1
