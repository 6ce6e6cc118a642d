timeout 100 python scripts/stall_probe.py 2000 2000 24 50 | tail -1
timeout 100 python scripts/stall_probe.py 3100 2600 24 50 | tail -1
for lib in "" paper_1307_2560_b200/libychg_b200_w4s3_p_alu.so paper_1307_2560_b200/libychg_b200_w4s2.so; do
  echo "=== lib ${lib:-default}"
  YCHG_LIB=$lib timeout 300 python scripts/pipe_timeline.py 21000 hbands 2>&1 | grep -E "isolated|graph|k=|finish phases" | head -4
  YCHG_LIB=$lib timeout 300 python scripts/pipe_timeline.py 21000 random 2>&1 | grep -E "isolated|graph|k=" | head -4
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline.py -q -m gpu -x 2>&1 | tail -2
