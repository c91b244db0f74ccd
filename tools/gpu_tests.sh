#!/bin/bash
# the whole GPU suite (optionally minus one test id) + smoke
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
DESEL=${2:+--deselect $2}
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 $DESEL > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
