set -x
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python scripts/pipe_timeline.py 21000 hbands "" 10 2>&1 | tail -30
timeout 300 python scripts/pipe_timeline.py 21000 random "" 2>&1 | tail -30
timeout 200 python scripts/pipe_timeline.py 2000 hbands 2>&1 | tail -8
