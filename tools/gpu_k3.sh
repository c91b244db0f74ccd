timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3
timeout 300 python bench.py --quick --steps 10 --warmup 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'], d['clocks'])"
