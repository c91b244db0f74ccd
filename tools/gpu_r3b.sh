#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 120 ./tools/gridbar_probe > $O/gridbar.txt 2>&1
bash tools/c2_variants.sh $1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 --deselect "tests/test_gpu_configs.py::test_single_chain_bench_launch_vs_oracle[c5]" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
