set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for w in gen k3 k1 f64; do timeout 120 python tools/probe.py $w 2>&1 | tail -12; echo "exit $w: $?"; done
