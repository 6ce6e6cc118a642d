for lib in "" paper_1307_2560_b200/libychg_b200_w4s4.so paper_1307_2560_b200/libychg_b200_w4s5.so "paper_1307_2560_b200/libychg_b200_w4s3_warps_links=8.so"; do
  echo "=== lib ${lib:-default}"
  YCHG_LIB=$lib timeout 300 python scripts/pipe_timeline.py 21000 hbands 2>&1 | grep -E "isolated|graph|k="
  YCHG_LIB=$lib timeout 300 python scripts/pipe_timeline.py 21000 random 2>&1 | grep -E "isolated|graph|k="
done
for i in 1 2 3; do ./oracle/_ref/acceptance_dropin 5; done
