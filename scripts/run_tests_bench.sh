set -x
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -3 | cut -c1-1500
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --pattern random 2>&1 | tail -3 | cut -c1-1200
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --counts-only 2>&1 | tail -3 | cut -c1-1200
