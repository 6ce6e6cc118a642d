L=paper_1307_2560_b200/libychg_b200.so
echo default; timeout 100 python scripts/host_counts_probe.py $L
echo direct16; YCHG_PAGEABLE_DIRECT_MB=16 timeout 100 python scripts/host_counts_probe.py $L
echo threads1; YCHG_COPY_THREADS=1 timeout 100 python scripts/host_counts_probe.py $L
echo threads8; YCHG_COPY_THREADS=8 timeout 100 python scripts/host_counts_probe.py $L
echo stage1; YCHG_STAGE_MB=1 timeout 100 python scripts/host_counts_probe.py $L
nproc; lscpu | grep -E "Model name|Socket|NUMA node\(s\)|^CPU\(s\)"
for v in "" 16; do echo "crit5 direct=$v"; YCHG_PAGEABLE_DIRECT_MB=$v ./oracle/_ref/acceptance_dropin 5; done
