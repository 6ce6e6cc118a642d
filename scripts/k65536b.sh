run() { env "$@" python bench.py --size 65536 --no-cpu-baseline --no-e2e --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', d['config']['plan'], round(d['ms_per_step']*1e3,2), 'us frac', d['roofline']['frac'], '| subset', round(d['north_star_subset']['ms_per_step']*1e3,2), d['north_star_subset']['roofline_frac'])"; }
run YCHG_SEGMENTS=2
run YCHG_SEGMENTS=4 YCHG_GRID=148
run YCHG_SEGMENTS=4
run YCHG_SEGMENTS=6 YCHG_GRID=148
run YCHG_SEGMENTS=8 YCHG_GRID=148
