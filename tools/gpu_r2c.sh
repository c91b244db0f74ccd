#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r2c; mkdir -p $O
timeout 120 ./tools/i8_probe > $O/i8_probe.txt 2>&1; echo "rc=$?" >> $O/i8_probe.txt
timeout 300 python tools/pageable_probe.py > $O/pageable_probe.txt 2>&1; echo "rc=$?" >> $O/pageable_probe.txt
timeout 900 python -m pytest tests/test_gpu_faults.py tests/test_gpu_parity.py -m gpu -q -rs --timeout 600 -k "fault or router or pageable or table or splitmix or chain_bitwise or cache or validation" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
