timeout 100 python scripts/stall_probe.py 2000 2000 24 50 | tail -1
timeout 100 python scripts/stall_probe.py 3100 2600 24 50 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/pipe_timeline.py 21000 hbands "" 5 4 2>&1 | grep -v "K=100 scan\|K=20 scan"
timeout 300 python scripts/pipe_timeline.py 21000 random "" 4 2>&1 | grep -v "K=100 scan\|K=20 scan"
