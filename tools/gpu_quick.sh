# tests + bench (no ncu)
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -4
timeout 600 python bench.py --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','matrices_per_s')}, d['roofline']['frac'], d['clocks'], d.get('e2e',{}).get('value'))"
