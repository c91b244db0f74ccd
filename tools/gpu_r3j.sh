#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
