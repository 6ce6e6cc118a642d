B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --pattern random"
export YCHG_LIB=paper_1307_2560_b200/libychg_b200_w8s4_compute_only.so
$B > gpurun_out/plainc.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ychg_scan_kernel -s 3 -c 1 -o gpurun_out/prof_compute $B > gpurun_out/ncu_c.log 2>&1
tail -1 gpurun_out/ncu_c.log
