#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 300 python tools/c2_once.py c2 3 > $O/c2_hash.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_faults.py -m gpu -q -k "k1h or chain or config2 or c2 or fault or history or large_chain" --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
bash tools/c2_variants.sh $1
