for k in "" 7; do for st in 20 50 100; do
  YCHG_SEGMENTS=$k python bench.py --no-cpu-baseline --no-e2e --steps $st 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('k', d['config']['plan']['seg_per_strip'], 'K', d['steps'], round(d['ms_per_step']*1e3,2), 'us frac', d['roofline']['frac'], '| subset', round(d['north_star_subset']['ms_per_step']*1e3,2), d['north_star_subset']['roofline_frac'])"
done; done
