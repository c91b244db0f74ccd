#!/bin/bash
# final round-2 profiles: ncu --set full of every product kernel on its bench
# workload, and the launch list of the default bench command
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on -f"
timeout 900 $NCU -k regex:k3h_batched -s 2 -c 1 -o $O/prof_k3h python bench.py --quick --steps 1 --warmup 2 > $O/ncu_k3h.log 2>&1
timeout 900 $NCU -k regex:k1p_gemm -s 12 -c 1 -o $O/prof_k1p python bench.py --workload c5 --quick --steps 1 --warmup 1 > $O/ncu_k1p.log 2>&1
timeout 600 $NCU -k regex:k1c_chain -s 1 -c 1 -o $O/prof_k1c python tools/c2_once.py c2 2 > $O/ncu_k1c.log 2>&1
timeout 900 $NCU -k regex:f64_gemm -s 10 -c 1 -o $O/prof_f64 python bench.py --workload c4 --quick --steps 1 --warmup 1 > $O/ncu_f64.log 2>&1
timeout 600 $NCU -k regex:k5i -s 3 -c 1 -o $O/prof_k5i python -c "
import sys; sys.path.insert(0,'.')
import bench, paper_1204_3052_b200 as mx
bench.run_mod(mx.Engine(0), n=4096, k=5, steps=1)" > $O/ncu_k5i.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --quick --steps 3 --warmup 3 > $O/launches_bench.log 2>&1
ls -la $O
