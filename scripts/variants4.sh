for lib in libychg_b200.so libychg_b200_w8s2_no_head.so libychg_b200_w8s2_compute_only.so; do
  for pat in hbands random; do
      r=$(YCHG_LIB=paper_1307_2560_b200/$lib timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --pattern $pat 2>&1 | tail -1)
      python - "$lib" "$pat" "$r" <<'PY'
import json, sys
lib, pat, r = sys.argv[1:]
try:
    d = json.loads(r)
    print(f"{lib:34s} {pat:7s} step {d['ms_per_step']*1000:7.2f} us  frac {d['roofline']['frac']:.3f}  HE {d['totals']['hyperedges']}")
except Exception as e:
    print(lib, pat, "FAILED", r[-300:])
PY
  done
done
