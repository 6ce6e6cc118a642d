# segments-per-strip sweep at 21000^2, K=100 steady state (full path and K1+K2 subset)
for k in ${KS:-2 3 4 2 3 4}; do
  r=$(YCHG_SEGMENTS=$k timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1)
  python - "$k" "$r" <<'PY'
import json, sys
k, r = sys.argv[1:]
try:
    d = json.loads(r)
    print(f"k={k} grid={d['config']['plan']['grid']} full {d['ms_per_step']*1000:6.2f} us frac {d['roofline']['frac']:.3f} | subset {d['north_star_subset']['ms_per_step']*1000:6.2f} us  eager {d['eager_launch_ms']*1000:6.1f} us")
except Exception as e:
    print(k, "FAILED", r[-300:])
PY
done
