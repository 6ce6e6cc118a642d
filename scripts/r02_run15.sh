timeout 100 python scripts/stall_probe.py 3100 2600 24 50 | tail -1
timeout 600 python bench.py 2>&1 | tail -1
timeout 600 python bench.py --pattern random --no-e2e 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
