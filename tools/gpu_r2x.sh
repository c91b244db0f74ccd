#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -k "cancellation or fixup or small_n or config1 or c1 or graph or zero or structured or batched" --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/c1_variants.sh $1
