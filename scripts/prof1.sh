set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --counts-only | cut -c1-900
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --pattern random | cut -c1-900
$B > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ychg_scan_kernel -s 4 -c 1 -o gpurun_out/prof_scan $B > gpurun_out/ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ychg_finish_kernel -s 4 -c 1 -o gpurun_out/prof_finish $B > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
