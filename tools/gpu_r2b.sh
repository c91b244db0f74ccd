#!/bin/bash
# round 2, session B: GPU suite after the cleanup, bench (incl. pageable e2e,
# in-kernel clock), 2 ranks sharing the GPU, K3H ncu capture
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 -s > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-extras > $O/bench_share2.json 2> $O/bench_share2.err
echo "share2 rc=$?" >> $O/bench_share2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --quick --steps 3 --warmup 1 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3h -s 2 -c 1 -o $O/prof_k3h python bench.py --quick --steps 1 --warmup 2 > $O/ncu_k3h.log 2>&1
echo "ncu rc=$?" >> $O/ncu_k3h.log
