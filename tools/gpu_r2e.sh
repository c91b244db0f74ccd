#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py -m gpu -q -rs --timeout 600 -k "modular or fault" > $O/pytest_mod.log 2>&1; echo "rc=$?" >> $O/pytest_mod.log
timeout 600 python - > $O/mod_bench.txt 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
import torch, bench, paper_1204_3052_b200 as mx
eng = mx.Engine(0)
for n in (1024, 2048, 4096, 8192):
    r = bench.run_mod(eng, n=n, k=257)
    print(json.dumps(r))
PY
echo "rc=$?" >> $O/mod_bench.txt
