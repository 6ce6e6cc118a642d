run() { lib=$1; shift; env "$@" YCHG_LIB=paper_1307_2560_b200/$lib python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $*', d['config']['plan']['grid'], round(d['ms_per_step']*1e3,2), d['roofline']['frac'], '| subset', round(d['north_star_subset']['ms_per_step']*1e3,2), d['north_star_subset']['roofline_frac'])"; }
for rep in 1 2; do
run libychg_b200.so
run libychg_b200_w8s4.so
done
