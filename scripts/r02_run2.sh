set -x
timeout 300 python scripts/pipe_timeline.py 21000 hbands "" 10 4 2>&1 | tail -30
timeout 200 python scripts/pipe_timeline.py 2000 hbands 2>&1 | tail -8
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "skip or pipelined or timing or column or profile" 2>&1 | tail -5
