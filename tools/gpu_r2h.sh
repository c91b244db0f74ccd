#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py -m gpu -q -rs --timeout 600 -s > $O/pytest_fused.log 2>&1; echo "rc=$?" >> $O/pytest_fused.log
