#!/bin/bash
# final-build profiles: the bench command's launch list (default workload, no
# secondary configs), one ncu --set full of K3H (the headline kernel) and of
# C2's K1C chain
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-extras --quick > $O/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3h_batched -s 3 -c 1 -o $O/k3h_full \
  python tools/c3_time.py 65536 2 > $O/k3h_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1c_chain -s 2 -c 1 -o $O/k1c_full \
  python tools/c2_once.py > $O/k1c_full.log 2>&1
