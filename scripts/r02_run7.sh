timeout 300 python scripts/host_counts_probe.py paper_1307_2560_b200/libychg_b200_r1.so paper_1307_2560_b200/libychg_b200.so paper_1307_2560_b200/libychg_b200_r1.so paper_1307_2560_b200/libychg_b200.so
YCHG_HOST_TIMING=1 timeout 100 python scripts/host_counts_probe.py paper_1307_2560_b200/libychg_b200.so 2>&1 | tail -20
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
