# segments-per-strip sweep at 21000^2 (grid = min(2*SMs, segments))
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o /tmp/block_tput scripts/micro/block_tput.cu && /tmp/block_tput
for k in "" 6 7 8 14 21 28; do
  r=$(YCHG_SEGMENTS=$k timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1)
  python - "$k" "$r" <<'PY'
import json, sys
k, r = sys.argv[1:]
try:
    d = json.loads(r)
    print(f"k={k or 'auto':5s} step {d['ms_per_step']*1000:7.2f} us  eager {d.get('eager_launch_ms',0)*1000:7.2f} us frac {d['roofline']['frac']:.3f}  HE {d['totals']['hyperedges']}")
except Exception as e:
    print(k, "FAILED", r[-300:])
PY
done
