#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py -m gpu -q -rs --timeout 600 -k "modular or fault" > $O/pytest_mod.log 2>&1; echo "rc=$?" >> $O/pytest_mod.log
timeout 600 python - > $O/mod_bench.txt 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
import torch, bench, paper_1204_3052_b200 as mx
eng = mx.Engine(0)
for n in (1024, 2048, 4096, 8192):
    r = bench.run_mod(eng, n=n, k=257)
    print(json.dumps(r))
print("int8 peak", bench.int8_peak_tops(torch.device("cuda", 0)))
PY
echo "rc=$?" >> $O/mod_bench.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k5i -s 3 -c 1 -o $O/prof_k5i python -c "
import sys; sys.path.insert(0,'.')
import bench, paper_1204_3052_b200 as mx
bench.run_mod(mx.Engine(0), n=4096, k=5, steps=1)" > $O/ncu_k5i.log 2>&1; echo "rc=$?" >> $O/ncu_k5i.log
