timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3
for w in c2 c5; do timeout 300 python bench.py --workload $w --quick --steps 5 --warmup 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['gpu_launches'])"; done
timeout 120 python tools/probe.py k1 2>&1 | tail -4
