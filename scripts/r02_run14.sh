timeout 100 python scripts/stall_probe.py 3100 2600 24 50 | tail -1
for pat in random hbands checker; do for k in "" 4; do YCHG_SEGMENTS=$k timeout 120 python scripts/ab_graph.py 21000 $pat; done; done
YCHG_NO_SKIP=1 timeout 120 python scripts/ab_graph.py 21000 random
timeout 900 python -m pytest tests -q -m gpu -x -k "skip or baseline or pipelined" 2>&1 | tail -2
