# round-2 first GPU pass: isolated latency, K=20 bench variants, GPU test suite
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 python scripts/isolated_scan_probe.py 21000 hbands 2>&1 | tail -8
timeout 120 python scripts/isolated_scan_probe.py 21000 random 2>&1 | tail -8
timeout 120 python scripts/isolated_scan_probe.py 2000 hbands 2>&1 | tail -8
for pat in hbands random; do
  timeout 180 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --pattern $pat 2>&1 | tail -2 | cut -c1-900
  YCHG_NO_SKIP=1 timeout 180 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --pattern $pat 2>&1 | tail -2 | cut -c1-900
  timeout 180 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --pattern $pat 2>&1 | tail -2 | cut -c1-900
done
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
