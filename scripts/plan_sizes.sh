# steady-state per-scan time by size with the current planner (K=100 graph)
for s in 8000 12000 16000 21000 32768 65536; do
  python bench.py --size $s --no-cpu-baseline --no-e2e --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['plan'], round(d['ms_per_step']*1e3,2), 'us frac', d['roofline']['frac'], '| subset', d['north_star_subset']['ms_per_step']*1e3, 'eager', d['eager_launch_ms']*1e3)"
done
