#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 900 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-extras --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err
