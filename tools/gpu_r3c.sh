#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 60 ./tools/k1c_trace 512 > $O/trace_push.txt 2>&1
timeout 60 ./tools/k1c_trace_pull 512 > $O/trace_pull.txt 2>&1
bash tools/c2_variants.sh $1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q --timeout 600 -k "k1c or K1C or one_launch or c2 or structured or edge" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
