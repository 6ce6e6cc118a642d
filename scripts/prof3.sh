B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain3.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ychg_scan_kernel -s 3 -c 1 -o gpurun_out/prof_v3 $B > gpurun_out/ncu_v3.log 2>&1
tail -2 gpurun_out/ncu_v3.log
