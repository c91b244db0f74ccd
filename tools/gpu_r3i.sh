#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
bash tools/c2_variants.sh $1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_faults.py -m gpu -q --timeout 600 -k "k1c or K1C or one_launch or c2 or structured or edge or fault or chain" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
