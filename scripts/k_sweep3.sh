run() { env "$@" python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', d['config']['plan']['grid'], round(d['ms_per_step']*1e3,2), d['roofline']['frac'], '| subset', round(d['north_star_subset']['ms_per_step']*1e3,2), d['north_star_subset']['roofline_frac'])"; }
for rep in 1 2; do
run YCHG_SEGMENTS=3
run YCHG_SEGMENTS=4
run YCHG_SEGMENTS=5
run YCHG_SEGMENTS=6
done
