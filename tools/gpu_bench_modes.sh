#!/bin/bash
# reference arm and the two-rank (shared GPU) path of bench.py
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_share2.json 2> $O/bench_share2.err; echo "rc=$?" >> $O/bench_share2.err
