for lib in libychg_b200.so libychg_b200_w8s2.so libychg_b200_w6s3.so libychg_b200_w4s4.so; do
  for pat in hbands random; do
    for extra in "" "--counts-only"; do
      r=$(YCHG_LIB=paper_1307_2560_b200/$lib timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --pattern $pat $extra 2>&1 | tail -1)
      python - "$lib" "$pat" "$extra" "$r" <<'PY'
import json, sys
lib, pat, extra, r = sys.argv[1:]
try:
    d = json.loads(r)
    print(f"{lib:26s} {pat:7s} {extra or 'full':13s} step {d['ms_per_step']*1000:7.2f} us  eager {d['eager_launch_ms']*1000:7.2f} us  frac {d['roofline']['frac']:.3f}  HE {d['totals']['hyperedges']}")
except Exception as e:
    print(lib, pat, extra, "FAILED", r[-300:])
PY
    done
  done
done
