#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 300 python tools/c2_once.py c2 3 > $O/c2_hash.txt 2>&1
bash tools/c2_variants.sh $1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "chain or multiply or c2 or config2 or gemm_rows" --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
