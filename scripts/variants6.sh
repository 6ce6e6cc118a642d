# L2 prefetch depth (YCHG_PREFETCH) variants; steps 5 and 30 (isolated-ish vs pipelined)
for lib in libychg_b200.so "libychg_b200_w8s2_prefetch=0.so" "libychg_b200_w8s2_prefetch=4.so"; do
  for st in 5 30; do
    for extra in "" "--counts-only"; do
      r=$(YCHG_LIB=paper_1307_2560_b200/$lib timeout 120 python bench.py --steps $st --warmup 5 --no-cpu-baseline --no-e2e $extra 2>&1 | tail -1)
      python - "$lib" "$st" "$extra" "$r" <<'PY'
import json, sys
lib, st, extra, r = sys.argv[1:]
try:
    d = json.loads(r)
    print(f"{lib:34s} steps {st:3s} {extra or 'full':13s} step {d['ms_per_step']*1000:7.2f} us eager {d.get('eager_launch_ms',0)*1000:7.2f} us frac {d['roofline']['frac']:.3f}")
except Exception as e:
    print(lib, st, extra, "FAILED", r[-300:])
PY
    done
  done
done
