timeout 60 python tools/probe.py acc 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -25
