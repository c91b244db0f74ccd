for w in diag k3 k1; do timeout 120 python tools/probe.py $w 2>&1 | tail -30; done
