for env in "YCHG_COOPERATIVE=0" "YCHG_COOPERATIVE=1"; do
  for pat in hbands random; do
    for extra in "" "--counts-only"; do
      r=$(env $env timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --pattern $pat $extra 2>&1 | tail -1)
      python - "$env" "$pat" "$extra" "$r" <<'PY'
import json, sys
lib, pat, extra, r = sys.argv[1:]
try:
    d = json.loads(r)
    print(f"{lib:20s} {pat:7s} {extra or 'full':13s} step {d['ms_per_step']*1000:7.2f} us  eager {d['eager_launch_ms']*1000:7.2f} us  frac {d['roofline']['frac']:.3f}  HE {d['totals']['hyperedges']}")
except Exception as e:
    print(lib, pat, extra, "FAILED", r[-600:])
PY
    done
  done
done
