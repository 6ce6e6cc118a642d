B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ychg_scan_kernel -s 3 -c 1 -o gpurun_out/prof_fused $B > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
