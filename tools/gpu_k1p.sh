timeout 120 python tools/probe.py k1 2>&1 | tail -5
timeout 120 python tools/probe.py acc 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -6
timeout 300 python bench.py --workload c5 --quick --steps 3 --warmup 1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'], d['ms_per_step'])"
